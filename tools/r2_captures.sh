#!/bin/bash
# full ncu captures (one launch each) of k_sample / k_big on C5 and C4 for the final round-2 evidence,
# then a C5 A/B of any libgirg_m_*.so variants present
cd $GRAFT_REPO_ROOT
for c in C5 C4; do
  for k in k_sample k_big; do
    timeout 900 ncu --set full --clock-control none --import-source on -k $k -c 1 -o /tmp/ev3_${c}_${k} -f \
      python tools/prof_one.py $c merged 1 nostats > gpurun_out/ev3_ncu_${c}_${k}.log 2>&1
    ncu -i /tmp/ev3_${c}_${k}.ncu-rep --page raw --csv > gpurun_out/ev3_raw_${c}_${k}.csv 2>&1
    ncu -i /tmp/ev3_${c}_${k}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ev3_src_${c}_${k}.csv 2>&1
    python tools/ncu_regions.py /tmp/ev3_src_${c}_${k}.csv > gpurun_out/ev3_regions_${c}_${k}.txt 2>&1
    gzip -c /tmp/ev3_src_${c}_${k}.csv > gpurun_out/ev3_src_${c}_${k}.csv.gz
  done
done
REPS=2 CFGS="C5" bash tools/ab_gpu.sh > /dev/null 2>&1; cat gpurun_out/sweep.log
