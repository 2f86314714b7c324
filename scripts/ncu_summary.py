"""Summarise ncu reports / launch lists into profiles/ (text + json)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        stalls = {}
        for i, n in enumerate(h):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_share_pct"] = {k: round(100 * v / tot, 1) for k, v in
                                sorted(stalls.items(), key=lambda x: -x[1]) if v / tot > 0.01}
        res.append(d)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        try:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
        except (ValueError, IndexError):
            pass
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "avg_ms": round(sum(v) / len(v) / 1e6, 4),
             "share_pct": round(100 * sum(v) / tot, 2)} for k, v in
            sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    data = raw(src) if mode == "rep" else launches(src)
    json.dump(data, open(dst, "w"), indent=1)
    print(json.dumps(data, indent=1)[:3000])
