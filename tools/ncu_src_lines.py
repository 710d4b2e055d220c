import csv, sys, collections
path = sys.argv[1]
rows = list(csv.reader(open(path)))
cur_file = None; hdr = None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr): continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    def g(name):
        i = hdr.index(name)
        try: return float(r[i])
        except: return 0.0
    ex = g("L1 Wavefronts Shared Excessive"); wf = g("L1 Wavefronts Shared"); st = g("Warp Stall Sampling (All Samples)")
    key = (cur_file.split("/")[-1], ln)
    a = agg[key]; a[0] += ex; a[1] += wf; a[2] += st; a[3] = r[1][:90]
tot_st = sum(v[2] for v in agg.values()) or 1
print("top excessive smem wavefronts (file:line  excess / total  stall%)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:15]:
    print(f"{k[0]}:{k[1]}  {v[0]:.0f} / {v[1]:.0f}  {100*v[2]/tot_st:.1f}%  {v[3]}")
print("top stall lines")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:20]:
    print(f"{k[0]}:{k[1]}  {100*v[2]/tot_st:.1f}%  smem {v[1]:.0f}  {v[3]}")
