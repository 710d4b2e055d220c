"""Summarise ncu reports (raw page) into a compact per-kernel table (JSON + stdout).

Usage: python tools/ncu_summary.py out.json report1.ncu-rep [report2.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time_us",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}
STALLS = ("barrier", "long_scoreboard", "short_scoreboard", "wait", "mio_throttle",
          "math_pipe_throttle", "not_selected", "lg_throttle", "branch_resolving")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for i, h in enumerate(hdr):
            if h in KEYS:
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                key = KEYS[h]
                if key in ("dram_read_B", "dram_write_B", "time_us"):
                    v *= SCALE.get(units[i], 1.0)
                d[key] = v
            for s in STALLS:
                if h == f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio":
                    try:
                        d["stall_" + s] = float(r[i])
                    except ValueError:
                        pass
        res.append(d)
    return res


if __name__ == "__main__":
    allres = {}
    for rep in sys.argv[2:]:
        allres[rep.split("/")[-1]] = summarise(rep)
    json.dump(allres, open(sys.argv[1], "w"), indent=1)
    for rep, rs in allres.items():
        print("##", rep)
        for d in rs:
            print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()})
