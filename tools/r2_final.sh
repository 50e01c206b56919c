#!/bin/bash
# final round-2 validation on the committed code: GPU suite, smoke, bench lines, T = 0 probe, Fig. 3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/fin_gputests.log 2>&1; tail -3 gpurun_out/fin_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; head -c 300 gpurun_out/fin_bench.json; echo
for c in C1 C2 C3 C4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/fin_cfg_$c.json 2> gpurun_out/fin_cfg_$c.err; done
timeout 300 python tools/t0_probe.py > gpurun_out/fin_t0.log 2>&1
timeout 600 python tools/fig3.py --reps 3 --out gpurun_out/fin_fig3.json > gpurun_out/fin_fig3.log 2>&1
timeout 600 python tools/batch_bench.py --B 64 --reps 5 --out gpurun_out/fin_batch_c1.json > gpurun_out/fin_batch.log 2>&1
timeout 900 python tools/hrg_bench.py > gpurun_out/fin_hrg.json 2> gpurun_out/fin_hrg.err
ls gpurun_out | grep fin_
