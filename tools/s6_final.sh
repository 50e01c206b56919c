#!/bin/bash
# final validation of the committed code (round 2, last session, final code): GPU suite, smoke, bench lines
# (default + per config + refined), reference arm, T = 0 probe, batch, HRG, C5 ncu launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/fin7_gputests.log 2>&1; tail -3 gpurun_out/fin7_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin7_smoke.log 2>&1; tail -1 gpurun_out/fin7_smoke.log
timeout 900 python bench.py > gpurun_out/fin7_bench.json 2> gpurun_out/fin7_bench.err; head -c 300 gpurun_out/fin7_bench.json; echo
for c in C1 C2 C3 C4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/fin7_cfg_$c.json 2> gpurun_out/fin7_cfg_$c.err; done
for c in C3 C5; do timeout 300 python bench.py --config $c --scheme refined --steps 5 --warmup 3 --no-cpu > gpurun_out/fin7_refined_$c.json 2> gpurun_out/fin7_refined_$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin7_ref.json 2> gpurun_out/fin7_ref.err; head -c 200 gpurun_out/fin7_ref.json; echo
timeout 300 python tools/t0_probe.py > gpurun_out/fin7_t0.log 2>&1
timeout 600 python tools/batch_bench.py --B 64 --reps 5 --out gpurun_out/fin7_batch_c1.json > gpurun_out/fin7_batch.log 2>&1
timeout 900 python tools/hrg_bench.py > gpurun_out/fin7_hrg.json 2> gpurun_out/fin7_hrg.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin7_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/fin7_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin7_launches_c5_refined.csv python bench.py --scheme refined --steps 2 --warmup 1 --no-cpu > gpurun_out/fin7_ncu_refined.log 2>&1
ls gpurun_out | grep fin7_
