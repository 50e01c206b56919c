# Source-level ncu captures of the sampling kernels (one launch each) for tools/ncu_lines.py.
# usage (on the GPU box): bash tools/prof_src.sh "C5 C4" "k_sample k_big"
set -x
cd $GRAFT_REPO_ROOT
CFGS=${1:-"C5 C4"}
KERNS=${2:-"k_sample k_big"}
SCHEME=${3:-merged}
mkdir -p gpurun_out
for cfg in $CFGS; do
  for k in $KERNS; do
    ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o /tmp/src_${cfg}_${k} -f python tools/prof_one.py $cfg $SCHEME 1 nostats > gpurun_out/ncu_${cfg}_${k}.log 2>&1
    ncu -i /tmp/src_${cfg}_${k}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_${cfg}_${k}.csv 2>&1
    python tools/ncu_lines.py /tmp/src_${cfg}_${k}.csv 60 > gpurun_out/lines_${cfg}_${k}.txt 2>&1
    ncu -i /tmp/src_${cfg}_${k}.ncu-rep --page raw --csv > gpurun_out/raw_${cfg}_${k}.csv 2>&1
    gzip -c /tmp/src_${cfg}_${k}.csv > gpurun_out/src_${cfg}_${k}.csv.gz
  done
done
ls -la gpurun_out
