cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "batch or smoke" > gpurun_out/gputest4.log 2>&1; tail -3 gpurun_out/gputest4.log
python tools/batch_bench.py --B 64 --reps 3 --out gpurun_out/batch_c1_r2.json 2>&1 | tail -4
python tools/batch_bench.py --B 16 --reps 3 --config C2 2>&1 | tail -3
