"""Summarise ncu --set full reports into a compact JSON/markdown for profiles/."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else rep}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = f"{vals[i]} {units[i]}".strip()
    stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(vals[i] or 0))
              for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    tot = sum(v for _, v in stalls) or 1.0
    d["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls, key=lambda x: -x[1])[:8]}
    return d


if __name__ == "__main__":
    res = [summarise(r) for r in sys.argv[1:]]
    print(json.dumps(res, indent=1))
