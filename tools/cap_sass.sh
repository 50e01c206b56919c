#!/bin/bash
# full capture + SASS-level source export of one sampling kernel:  C=C5 K=k_sample LIB=... tools/cap_sass.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
c=${C:-C5}; k=${K:-k_sample}; tag=${TAG:-cur}
GIRG_LIBRARY=${LIB:-paper_1905_06706_b200/libgirg.so} timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:$k -c 1 -o /tmp/cs_${tag}_$c -f python tools/prof_one.py $c merged 1 nostats > gpurun_out/cs_${tag}_$c.log 2>&1
ncu -i /tmp/cs_${tag}_$c.ncu-rep --page raw --csv > gpurun_out/cs_raw_${tag}_$c.csv 2>&1
ncu -i /tmp/cs_${tag}_$c.ncu-rep --page source --csv --print-source cuda,sass > /tmp/cs_src.csv 2>&1
gzip -c /tmp/cs_src.csv > gpurun_out/cs_src_${tag}_$c.csv.gz
tail -2 gpurun_out/cs_${tag}_$c.log
