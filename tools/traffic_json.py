"""profiles/ncu_traffic.json from ncu_summary JSONs of the box-solve passes:
DRAM read + write bytes per launch of each pass (transform-rows: rows_fwd_reg
/ rows_inv_reg, transform-cols: cols_tri / cols_reg), f64 and c128, and their
average over one bench step's launch mix (4 f64 launches per c128 launch pair,
the same weighting as bench.py's roofline `achieved`).

    python tools/traffic_json.py out.json summary1.json [summary2.json ...]
"""
import json
import sys

dst, srcs = sys.argv[1], sys.argv[2:]
acc = {"transform-rows": {"f64": [], "c128": []}, "transform-cols": {"f64": [], "c128": []},
       "diagonal-scale": {"f64": [], "c128": []}}
for src in srcs:
    for ks in json.load(open(src)).values():
        for k in ks:
            name = k["kernel"]
            if "rows_fwd_reg" in name or "rows_inv_reg" in name or "rows_fwd_facr" in name:
                pas = "transform-rows"
            elif "rows_odd_facr" in name:
                pas = "diagonal-scale"
            elif "cols_tri" in name or "cols_reg" in name:
                pas = "transform-cols"
            else:
                continue
            dt = "c128" if "<1," in name or "<(bool)1" in name or "<true" in name else "f64"
            acc[pas][dt].append(k["dram_read_B"] + k["dram_write_B"])
out = {"source": srcs}
for pas, d in acc.items():
    f = sum(d["f64"]) / len(d["f64"]) if d["f64"] else None
    c = sum(d["c128"]) / len(d["c128"]) if d["c128"] else None
    out[pas + ":f64"] = f
    out[pas + ":c128"] = c
    if f is not None and c is not None:
        out[pas] = (2 * f + c) / 3            # per bench step: 2 f64 solves per c128 solve
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out))
