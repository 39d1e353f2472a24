"""Summarise an ncu --set full report into the JSON kept under profiles/.

  python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/r02/x.json

One object per profiled launch, keyed by kernel kind (forward / adjoint /
epilogue / cta_adjoint / fused, from the kernel name), holding the metrics
DESIGN.md and the bench's roofline cite: duration, DRAM bytes, registers, grid,
occupancy, issue activity, FP64 pipe, cache hit rates, instructions and the
main stall reasons per issue.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
] + [f"smsp__average_warps_issue_stalled_{r}_per_issue_active.ratio"
     for r in ("barrier", "wait", "long_scoreboard", "short_scoreboard", "no_instruction", "math_pipe_throttle",
               "branch_resolving", "selected", "not_selected", "dispatch_stall", "mio_throttle", "lg_throttle")]


def kind(name: str) -> str:
    if "lane_adj" in name:
        return "adjoint"
    if "lane_epi" in name:
        return "epilogue"
    if "fwd_kernel" in name:
        return "forward"
    if "fused_kernel" in name:
        return "cta_adjoint" if ", 2" in name or "(int)2" in name else "fused"
    return name.split("(")[0].split()[-1]


def main(rep: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        rec = {"Kernel Name": name}
        for m in METRICS:
            if m in d:
                rec[m] = {"value": d[m], "unit": units[hdr.index(m)]}
        k = kind(name)
        key, n = k, 1
        while key in out:
            n += 1
            key = f"{k}#{n}"
        out[key] = rec
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
