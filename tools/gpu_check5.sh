cd $GRAFT_REPO_ROOT
for lib in paper_1905_06706_b200/libgirg.so paper_1905_06706_b200/libgirg_m_noload1.so paper_1905_06706_b200/libgirg_m_noload2.so; do
  for c in C2 C4 C5; do
    r=$(GIRG_LIBRARY=$lib timeout 120 python tools/prof_one.py $c merged 3 nostats 2>&1 | tail -1 | awk '{print $5}')
    echo "$(basename $lib) $c sample_ms=$r"
  done
done 2>&1 | tee gpurun_out/noload.log
# bounds-checked build (GIRG_DEBUG: every indexed access of the sampler checked, __trap on failure)
GIRG_LIBRARY=paper_1905_06706_b200/libgirg_debug.so timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "not C5 and not baseline_config" > gpurun_out/debug_tests.log 2>&1; tail -3 gpurun_out/debug_tests.log
