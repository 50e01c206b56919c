#!/bin/bash
# quick per-config timing (device-timed girg_edges, no oracle / e2e legs); writes gpurun_out/ball_<tag>_<cfg>.json
tag=${1:-cur}
for c in C1 C2 C3 C4 C5; do
  timeout 150 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ball_${tag}_$c.json 2> gpurun_out/ball_${tag}_$c.err
done
