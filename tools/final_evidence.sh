cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/fin_gputests.log 2>&1; tail -12 gpurun_out/fin_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; head -c 300 gpurun_out/fin_bench.json; echo
for c in C1 C2 C3 C4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/fin_cfg_$c.json 2> gpurun_out/fin_cfg_$c.err; done
timeout 600 python tools/fig3.py --reps 3 --out gpurun_out/fin_fig3.json > gpurun_out/fin_fig3.log 2>&1
timeout 900 python tools/shard_balance.py C3 C5 > gpurun_out/fin_shard_balance.json 2> gpurun_out/fin_shard_balance.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; head -c 300 gpurun_out/fin_ref.json
