#!/bin/bash
# T = 0 sampling times (tools/t0_probe.py) and C3/C5 sampling for every libgirg*.so variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in paper_1905_06706_b200/libgirg.so paper_1905_06706_b200/libgirg_m_*.so; do
  echo "== $(basename $lib)"
  GIRG_LIBRARY=$lib timeout 300 python tools/t0_probe.py 2>&1 | awk '{print $1, $2, $6, $7}'
  for c in ${CFGS:-C3 C5}; do
    r=$(GIRG_LIBRARY=$lib timeout 180 python tools/prof_one.py $c merged 2 nostats 2>&1 | tail -1 | awk '{print $5}')
    echo "$c sample_ms=$r"
  done
done 2>&1 | tee gpurun_out/ab_t0.log
