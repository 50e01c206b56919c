#!/bin/bash
# quick parity + sampling A/B of the library variants, then the sampling kernels' DRAM bytes on C5
cd $GRAFT_REPO_ROOT
REPS=${REPS:-2} CFGS=${CFGS:-"C2 C3 C4 C5"} bash tools/ab_gpu.sh > /dev/null 2>&1
tail -3 gpurun_out/qp.log; sort -k2,2 -k1,1 gpurun_out/sweep.log
for lib in paper_1905_06706_b200/libgirg.so paper_1905_06706_b200/libgirg_m_*.so; do
  GIRG_LIBRARY=$lib timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:"k_sample|k_big" --csv python tools/prof_one.py C5 merged 1 nostats 2>/dev/null | grep '^"' > gpurun_out/traffic_$(basename $lib .so).csv
  echo "== $(basename $lib)"; grep -v "Metric Name" gpurun_out/traffic_$(basename $lib .so).csv | awk -F'","' '{print $5, $13, $15}' | sed 's/"//g'
done
