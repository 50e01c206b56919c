# compute-sanitizer runs (memcheck, racecheck, synccheck) of the sampling kernels on small configs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  for cfg in C1 C2 C3; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_one.py $cfg > gpurun_out/sanitizer/${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -c 'ERROR SUMMARY' gpurun_out/sanitizer/${tool}_${cfg}.log) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitizer/${tool}_${cfg}.log | tail -1)"
  done
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_one.py batch > gpurun_out/sanitizer/${tool}_batch.log 2>&1
  echo "$tool batch rc=$? $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitizer/${tool}_batch.log | tail -1)"
done
