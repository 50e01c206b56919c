cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "scale or smoke or C1 or batch" > gpurun_out/gputest3.log 2>&1; tail -3 gpurun_out/gputest3.log
python tools/fig3.py --reps 3 --out gpurun_out/fig3_r2.json > gpurun_out/fig3_r2.log 2>&1; python - <<'PY'
import json
for r in json.load(open("gpurun_out/fig3_r2.json"))["rows"] if isinstance(json.load(open("gpurun_out/fig3_r2.json")), dict) else json.load(open("gpurun_out/fig3_r2.json")):
    print(r["n"], r["d"], r["T"], "weights %.3f scale %.3f pre %.3f edges %.3f ms" % (r["ms"]["weights"], r["ms"]["scale"], r["ms"]["pre"], r["ms"]["edges"]))
PY
