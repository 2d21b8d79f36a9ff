"""Condense an .ncu-rep (--set full) into the JSON kept under profiles/:
per kernel launch: duration, DRAM bytes / throughput, DMMA / FP64 pipe
activity, registers, occupancy, bank conflicts, and the warp-stall breakdown.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [kernel-regex]
"""
import csv
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
]


def summarize(rep, rx=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    rows = list(csv.reader(out))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "")
        if rx and not re.search(rx, name):
            continue
        k = {"kernel": name}
        for key in KEYS:
            if key in d and d[key] != "":
                k[key] = f"{d[key]} {u.get(key, '')}".strip()
        st = {key.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
              for key, v in d.items()
              if key.startswith("smsp__pcsamp_warps_issue_stalled_") and not key.endswith(
                  "not_issued") and v not in ("", "0")}
        tot = sum(st.values()) or 1.0
        k["warp_stall_share"] = {kk: round(v / tot, 3)
                                 for kk, v in sorted(st.items(), key=lambda x: -x[1])[:10]}
        res.append(k)
    return res


if __name__ == "__main__":
    res = summarize(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 else None)
    json.dump({"report": sys.argv[1].split("/")[-1], "launches": res}, open(sys.argv[2], "w"),
              indent=1)
    print(json.dumps(res, indent=1)[:3000])
