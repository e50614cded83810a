"""Summarise an `ncu --set full` report of the hot kernels into the JSON that
bench.py reads `roofline.traffic` from (profiles/r2_ncu_summary.json).

  python tools/ncu_summarize.py REPORT.ncu-rep OUT.json

Per kernel launch: duration, DRAM bytes read/written, pipe utilisation (XU =
MUFU, FMA), issue/warps active, registers, grid, SM clock, the top stall
reasons, and the FP32/XU instruction counts (the E-step's instruction mix
from hardware counters: FP32 lane-ops = 2·(FFMA2 + FADD2 + FMUL2) + FFMA +
FADD + FMUL thread instructions; MUFU lane-ops = 32 · XU warp instructions).
"""
import csv
import io
import json
import subprocess
import sys


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}

    def get(r, name):
        i = idx.get(name)
        return num(r[i]) if i is not None and i < len(r) else None

    kernels = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        name = r[idx["Kernel Name"]].split("(")[0]
        dur_ms = get(r, "gpu__time_duration.sum")  # ncu reports ms for these launches
        unit = rows[1][idx["gpu__time_duration.sum"]]
        time_us = dur_ms * (1e3 if unit == "ms" else 1e-3 if unit == "ns" else 1.0)
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = get(r, "dram__bytes_read.sum") * scale.get(rows[1][idx["dram__bytes_read.sum"]], 1.0)
        wr = get(r, "dram__bytes_write.sum") * scale.get(rows[1][idx["dram__bytes_write.sum"]], 1.0)
        stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""): get(r, h) for h in idx
            if h.startswith("smsp__average_warps_issue_stalled_")
            and h.endswith("_per_issue_active.ratio")}
        top = dict(sorted(((k, v) for k, v in stalls.items() if v), key=lambda kv: -kv[1])[:5])
        op = {k: get(r, f"sm__sass_thread_inst_executed_op_{k}_pred_on.sum")
              for k in ("ffma2", "fadd2", "fmul2", "ffma", "fadd", "fmul")}
        xu = get(r, "sm__inst_executed_pipe_xu.sum")
        fp32_lane_ops = None
        if all(v is not None for v in op.values()):
            fp32_lane_ops = 2 * (op["ffma2"] + op["fadd2"] + op["fmul2"]) + op["ffma"] + \
                op["fadd"] + op["fmul"]
        kernels.append({
            "kernel": name, "time_us": time_us, "dram_read_B": rd, "dram_write_B": wr,
            "dram_pct_peak": get(r, "dram__throughput.avg.pct_of_peak_sustained_elapsed")
            or get(r, "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "xu_pipe_pct": get(r, "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": get(r, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": get(r, "sm__issue_active.avg.pct_of_peak_sustained_active")
            or get(r, "sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
            "warps_active_pct": get(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "regs": get(r, "launch__registers_per_thread"), "grid": get(r, "launch__grid_size"),
            "sm_clock_hz": (get(r, "sm__cycles_elapsed.avg.per_second") or 0) * 1e9,
            "top_stalls_per_issue": top,
            "fp32_thread_inst": op, "fp32_lane_ops": fp32_lane_ops,
            "xu_warp_inst": xu, "mufu_lane_ops": xu * 32 if xu is not None else None,
        })
    colsum = [k["dram_read_B"] + k["dram_write_B"] for k in kernels
              if k["kernel"].endswith("colsum_bulk_kernel")]
    json.dump({"report": rep, "kernels": kernels,
               "colsum_dram_bytes_per_launch": sum(colsum) / len(colsum) if colsum else None},
              open(out, "w"), indent=1)
    for k in kernels:
        print(f"{k['kernel'][:40]:40s} {k['time_us']:10.1f} us  DRAM {(k['dram_read_B'] + k['dram_write_B']) / 1e6:8.1f} MB"
              f"  XU {k['xu_pipe_pct'] or 0:5.1f}%  FMA {k['fma_pipe_pct'] or 0:5.1f}%")


if __name__ == "__main__":
    main()
