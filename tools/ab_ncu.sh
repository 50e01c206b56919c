#!/bin/bash
# per-kernel duration / instructions / warp-state stalls of the sampling kernels for each library
# variant (and optional env settings):  C=C3 tools/ab_ncu.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
c=${C:-C3}
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 900 ncu --clock-control none --section WarpStateStats --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_ld.sum \
    -k regex:"k_sample|k_big" --csv python tools/prof_one.py $c merged 1 nostats > gpurun_out/abn_${c}_$tag.csv 2> gpurun_out/abn_${c}_$tag.err
}
run base GIRG_LIBRARY=paper_1905_06706_b200/libgirg_m_base.so
run new GIRG_LIBRARY=paper_1905_06706_b200/libgirg.so
run new_big1 GIRG_LIBRARY=paper_1905_06706_b200/libgirg.so GIRG_BIG1=0
for f in gpurun_out/abn_${c}_*.csv; do
  echo "== $f"
  python - "$f" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
for r in rows[1:]:
    m = r[im]
    if m in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_ld.sum") or "Stall" in m or "stall" in m:
        try:
            if float(r[iv].replace(",", "")) == 0: continue
        except ValueError:
            pass
        print(r[ik][:28], m[:60], r[iv])
PY
done
