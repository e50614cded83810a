"""Summarise an ncu --set full report (raw page) into profiles/*.json + text."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_B": "dram__bytes_read.sum",
    "dram_write_B": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
}


def to_float(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "us": 1, "ms": 1e3,
             "ns": 1e-3, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}
    return x * scale.get(unit, 1)


def main(rep, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(".ratio")]
    kernels = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for name, key in KEYS.items():
            if key in hdr:
                i = hdr.index(key)
                k[name] = to_float(r[i], units[i])
        stalls = sorted(((float(r[i] or 0), hdr[i].split("stalled_")[1].split("_per")[0])
                         for i in stall_cols), reverse=True)[:5]
        k["top_stalls_per_issue"] = {n: round(v, 3) for v, n in stalls}
        kernels.append(k)
    summary = {"report": rep, "kernels": kernels}
    cs = [k for k in kernels if k["kernel"].startswith("colsum")]
    if cs:
        summary["colsum_dram_bytes_per_launch"] = sum(
            k["dram_read_B"] + k["dram_write_B"] for k in cs) / len(cs)
    json.dump(summary, open(out_json, "w"), indent=1)
    for k in kernels:
        print(json.dumps(k))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
