cd $GRAFT_REPO_ROOT
c=${C:-C3}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample -c 1 -o /tmp/cap_$c -f \
  python tools/prof_one.py $c merged 1 nostats > gpurun_out/cap_$c.log 2>&1
ncu -i /tmp/cap_$c.ncu-rep --page raw --csv > gpurun_out/cap_raw_$c.csv 2>&1
ncu -i /tmp/cap_$c.ncu-rep --page source --csv --print-source cuda,sass > /tmp/cap_src_$c.csv 2>&1
python tools/ncu_lines.py /tmp/cap_src_$c.csv > gpurun_out/cap_lines_$c.txt 2>&1
gzip -c /tmp/cap_src_$c.csv > gpurun_out/cap_src_$c.csv.gz
tail -3 gpurun_out/cap_$c.log
