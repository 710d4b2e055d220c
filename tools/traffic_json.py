"""profiles/ncu_traffic.json from an ncu_summary JSON of the column-pass
captures: DRAM read + write bytes per launch of cols_reg, f64 and c128, and
their average over one bench step's launch mix (4 f64 + 2 c128 launches, the
same weighting as bench.py's roofline `achieved`).

    python tools/traffic_json.py prof_cols.json out.json
"""
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
d = json.load(open(src))
f64, c128 = [], []
for ks in d.values():
    for k in ks:
        if "cols_reg" not in k["kernel"]:
            continue
        b = k["dram_read_B"] + k["dram_write_B"]
        (c128 if "<1," in k["kernel"] else f64).append(b)
out = {"source": src, "f64_bytes_per_launch": sum(f64) / len(f64) if f64 else None,
       "c128_bytes_per_launch": sum(c128) / len(c128) if c128 else None}
if f64 and c128:
    out["cols_bytes_per_launch"] = (4 * out["f64_bytes_per_launch"] + 2 * out["c128_bytes_per_launch"]) / 6
elif f64:
    out["cols_bytes_per_launch"] = out["f64_bytes_per_launch"]
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out))
