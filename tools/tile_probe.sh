#!/bin/bash
# sampling time vs points per tile (GIRG_TILE_PTS) on C1 / C2 / C3, plus quick parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/quick_parity.py > gpurun_out/qp.log 2>&1; tail -1 gpurun_out/qp.log
for c in C1 C2 C3; do
  for ts in 32 16 8 4; do
    r=$(GIRG_TILE_PTS=$ts timeout 180 python tools/prof_one.py $c merged 5 nostats 2>&1 | tail -1 | awk '{print $5}')
    echo "$c tile_pts=$ts sample_ms=$r"
  done
done 2>&1 | tee gpurun_out/tile_probe.log
timeout 300 python tools/t0_probe.py 2>&1 | tail -1
