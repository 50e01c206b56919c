cd $GRAFT_REPO_ROOT
timeout 600 python tools/quick_parity.py > gpurun_out/qp.log 2>&1; tail -2 gpurun_out/qp.log
for lib in paper_1905_06706_b200/libgirg.so paper_1905_06706_b200/libgirg_m_*.so; do
  for c in ${CFGS:-C2 C3 C4 C5}; do
    r=$(GIRG_LIBRARY=$lib timeout 120 python tools/prof_one.py $c merged 3 nostats 2>&1 | tail -1 | awk '{print $5}')
    echo "$(basename $lib) $c sample_ms=$r"
  done
done 2>&1 | tee gpurun_out/sweep.log
