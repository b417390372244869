"""Summarise one kernel of an `ncu --set full` report into the profiles/ JSON layout (dev tool).

usage: python tools/ncu_full_summary.py report.ncu-rep "source note" [kernel-substring] > profiles/<name>.json
(the first profiled launch whose name contains the substring; default the first launch)
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum",
    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "launch__grid_size", "launch__block_size",
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main() -> None:
    rep, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    want = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    vals = next(r for r in rows[2:] if want in r[ik])
    d = {k: (v, u) for k, u, v in zip(hdr, units, vals)}
    metrics = {k: {"value": d[k][0], "unit": d[k][1]} for k in KEYS if k in d}
    stalls = {}
    for k, (v, _) in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    top = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    traffic = sum(float(d[k][0].replace(",", "")) * SCALE.get(d[k][1], 1.0)
                  for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in d)
    print(json.dumps({"source": note, "kernel": d.get("Kernel Name", ("?",))[0], "metrics": metrics,
                      "stall_reasons_pct": top, "traffic_bytes_per_launch": traffic}, indent=1))


if __name__ == "__main__":
    main()
