import json, glob, sys
for f in sorted(glob.glob(sys.argv[1])):
    try: d = json.load(open(f))
    except Exception as e: print(f, "ERR", e); continue
    for side in ("forward", "adjoint"):
        s = d[side]; sw = {k: v["ms"] for k, v in s["sweep"].items()}
        print(f"{f:28s} {side:7s} {sw} pos/nnz={s['padded_ratio']:.3f} slots/nnz={s['slots_per_nnz']:.4f}")
