#!/bin/bash
# full ncu captures (one launch each) of the final code's sampling kernels on C5: MERGED k_sample /
# k_big and REFINED k_big, raw pages + source-region summaries
cd $GRAFT_REPO_ROOT
for spec in merged:k_sample merged:k_big refined:k_big; do
  s=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/ev7_${s}_${k} -f \
    python tools/prof_one.py C5 $s 1 nostats > gpurun_out/ev7_ncu_${s}_${k}.log 2>&1
  ncu -i /tmp/ev7_${s}_${k}.ncu-rep --page raw --csv > gpurun_out/ev7_raw_C5_${s}_${k}.csv 2>&1
  ncu -i /tmp/ev7_${s}_${k}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ev7_src_${s}_${k}.csv 2>&1
  python tools/ncu_regions.py /tmp/ev7_src_${s}_${k}.csv > gpurun_out/ev7_regions_C5_${s}_${k}.txt 2>&1
  python tools/ncu_lines.py /tmp/ev7_src_${s}_${k}.csv 60 > gpurun_out/ev7_lines_C5_${s}_${k}.txt 2>&1
  tail -3 gpurun_out/ev7_ncu_${s}_${k}.log
done
ls -la gpurun_out | grep ev7_
