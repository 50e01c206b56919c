#!/bin/bash
# One GPU call producing the round's evidence (outputs in gpurun_out/ev2_*): bench line (C5 default),
# per-config lines, the C5 ncu launch list, full captures of both sampling kernels on C5 and C4,
# the batch and shard-balance tools, Fig. 3.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/ev2_bench.json 2> gpurun_out/ev2_bench.err
for c in C1 C2 C3 C4 C5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/ev2_cfg_$c.json 2> gpurun_out/ev2_cfg_$c.err
done
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev2_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ev2_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev2_ncu_launch.log 2>&1
for c in C5 C4; do
  for k in k_sample k_big; do
    timeout 900 ncu --set full --clock-control none --import-source on -k $k -c 1 -o /tmp/ev2_${c}_${k} -f \
      python tools/prof_one.py $c merged 1 nostats > gpurun_out/ev2_ncu_${c}_${k}.log 2>&1
    ncu -i /tmp/ev2_${c}_${k}.ncu-rep --page raw --csv > gpurun_out/ev2_raw_${c}_${k}.csv 2>&1
    ncu -i /tmp/ev2_${c}_${k}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ev2_src_${c}_${k}.csv 2>&1
    python tools/ncu_regions.py /tmp/ev2_src_${c}_${k}.csv > gpurun_out/ev2_regions_${c}_${k}.txt 2>&1
  done
done
timeout 600 python tools/batch_bench.py --B 64 --reps 5 --out gpurun_out/ev2_batch_c1.json > gpurun_out/ev2_batch.log 2>&1
timeout 900 python tools/shard_balance.py C3 C5 > gpurun_out/ev2_shard_balance.json 2> gpurun_out/ev2_shard_balance.err
timeout 900 python tools/fig3.py --reps 3 --out gpurun_out/ev2_fig3.json > gpurun_out/ev2_fig3.log 2>&1
ls -la gpurun_out | head -60
