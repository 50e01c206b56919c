#!/bin/bash
# time C2 / C4 sampling for every paper_1905_06706_b200/libgirg_<tag>.so variant
for lib in paper_1905_06706_b200/libgirg_m*.so; do
  for c in ${CFGS:-C2 C4}; do
    r=$(GIRG_LIBRARY=$lib timeout 90 python tools/prof_one.py $c merged 3 nostats 2>&1 | tail -1 | awk '{print $5}')
    echo "$(basename $lib) $c sample_ms=$r"
  done
done
