#!/bin/bash
# One GPU call producing the round's evidence: GPU tests, smoke, bench line, per-config bench,
# ncu launch list and full captures of the sampling kernels.  Outputs in gpurun_out/.
timeout 1500 python -u -m pytest tests -x -q -m gpu > gpurun_out/ev_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ev_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ev_smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
bash tools/bench_all.sh ev
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ev_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev_ncu_launch.log 2>&1
timeout 300 python tools/prof_one.py C5 merged 1 nostats > gpurun_out/ev_p5.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample -c 1 -o gpurun_out/ev_prof_c5 \
    python tools/prof_one.py C5 merged 1 nostats > gpurun_out/ev_ncu5.log 2>&1
timeout 300 python tools/prof_one.py C4 merged 1 nostats > gpurun_out/ev_p4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample -c 1 -o gpurun_out/ev_prof_c4 \
    python tools/prof_one.py C4 merged 1 nostats > gpurun_out/ev_ncu4.log 2>&1
