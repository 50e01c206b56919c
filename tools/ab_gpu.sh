#!/bin/bash
# GPU A/B: quick parity of the working library, then sampling-phase times of every libgirg*.so
# variant, interleaved per config:  CFGS="C2 C5" REPS=2 tools/ab_gpu.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/quick_parity.py --big > gpurun_out/qp.log 2>&1; tail -16 gpurun_out/qp.log
for rep in $(seq ${REPS:-1}); do
  for c in ${CFGS:-C1 C2 C3 C4 C5}; do
    for lib in paper_1905_06706_b200/libgirg.so paper_1905_06706_b200/libgirg_m_*.so; do
      r=$(GIRG_LIBRARY=$lib timeout 180 python tools/prof_one.py $c merged 3 nostats 2>&1 | tail -1 | awk '{print $5}')
      echo "$(basename $lib) $c sample_ms=$r"
    done
  done
done 2>&1 | tee gpurun_out/sweep.log
