# ncu full captures (one launch each) of the sampling kernels on C5 and C4 + source-region summaries
cd $GRAFT_REPO_ROOT
for c in C5 C4; do
  for k in k_sample k_big; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/ev2_${c}_${k} -f \
      python tools/prof_one.py $c merged 1 nostats > gpurun_out/ev2_ncu_${c}_${k}.log 2>&1
    ncu -i /tmp/ev2_${c}_${k}.ncu-rep --page raw --csv > gpurun_out/ev2_raw_${c}_${k}.csv 2>&1
    ncu -i /tmp/ev2_${c}_${k}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ev2_src_${c}_${k}.csv 2>&1
    python tools/ncu_regions.py /tmp/ev2_src_${c}_${k}.csv > gpurun_out/ev2_regions_${c}_${k}.txt 2>&1
  done
done
