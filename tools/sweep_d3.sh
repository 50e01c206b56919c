#!/bin/bash
for lib in paper_1905_06706_b200/libgirg_s*.so; do
  for bw in 4096 8192 32768; do
    r=$(GIRG_LIBRARY=$lib GIRG_BIG_WORK=$bw GIRG_ITEM_WORK=$((bw/2)) timeout 90 python tools/prof_one.py C5 merged 2 nostats 2>&1 | tail -1 | awk '{print $5}')
    r3=$(GIRG_LIBRARY=$lib GIRG_BIG_WORK=$bw GIRG_ITEM_WORK=$((bw/2)) timeout 90 python tools/prof_one.py C3 merged 2 nostats 2>&1 | tail -1 | awk '{print $5}')
    echo "$(basename $lib) bw=$bw C5 sample_ms=$r C3 sample_ms=$r3"
  done
done
