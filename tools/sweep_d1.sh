#!/bin/bash
# development sweep of the d = 1 knobs (task height G, job slots, big-job threshold)
for lib in paper_1905_06706_b200/libgirg_g*.so; do
  for bw in 256 512 2048; do
    for c in C2 C4; do
      r=$(GIRG_LIBRARY=$lib GIRG_BIG_WORK=$bw GIRG_ITEM_WORK=$((bw/2)) timeout 60 python tools/prof_one.py $c merged 3 nostats 2>&1 | tail -1 | awk '{print $5}')
      echo "$(basename $lib) bw=$bw $c sample_ms=$r"
    done
  done
done
