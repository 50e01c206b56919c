import glob, json, sys
for f in sorted(glob.glob(sys.argv[1])):
    try:
        j = json.load(open(f))
    except Exception:
        print(f, "no result"); continue
    r = j["roofline"]
    print(f"{j['config']['workload'][:36]:36s} {j['value']:.3g} e/s  {j['ms_per_step']:8.3f} ms  sample {r['phases_ms']['ms_sample']:8.3f}  index {r['phases_ms']['ms_index']:6.3f}  frac {r['frac']:.4f}")
