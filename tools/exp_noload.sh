cd $GRAFT_REPO_ROOT
for lib in paper_1905_06706_b200/libgirg.so paper_1905_06706_b200/libgirg_m_noload.so; do
  for c in C4 C5; do
    r=$(GIRG_LIBRARY=$lib timeout 120 python tools/prof_one.py $c merged 3 nostats 2>&1 | tail -1 | awk '{print $5}')
    echo "$(basename $lib) $c sample_ms=$r"
  done
done
# setup-only timing: jobs set up, units skipped (GIRG_DEV_FLAGS=1, profile build)
for c in C4 C5; do
  r=$(GIRG_DEV_FLAGS=1 GIRG_LIBRARY=paper_1905_06706_b200/libgirg_m_prof.so timeout 120 python tools/prof_one.py $c merged 3 nostats 2>&1 | tail -1 | awk '{print $5}')
  echo "setup-only $c sample_ms=$r"
done
