"""Per-instruction hot spots from an ncu report's SASS source page.

    python tools/ncu_src.py report.ncu-rep kernel_regex [top] [launch_skip]
Prints the instructions with the most stall samples and the shared-memory
instructions with excessive wavefronts (bank conflicts)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ix = {n: (h.index(n) if n in h else None)
      for n in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                "L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared", "Instructions Executed")}
data = rows[1:]
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
data = [r for r in data if r and r[0].startswith("0x")]
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"total stall samples {tot:.0f}")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    print(f"{f(r,'Warp Stall Sampling (All Samples)')/tot*100:5.1f}%  {r[ix['Source']].strip()[:80]}")
print("--- smem excessive wavefronts")
ex = sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))
for r in ex[:12]:
    if f(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"{f(r,'L1 Wavefronts Shared Excessive'):10.0f} / {f(r,'L1 Wavefronts Shared'):10.0f}  {r[ix['Address']]} {r[ix['Source']].strip()[:70]}")
