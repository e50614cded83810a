"""Copy a tools/gpu_round.sh result (gpurun_out/round/) into profiles/ as the
round's evidence: bench lines per workload, the reference arm, the parity
log, the ncu launch list and its per-kernel share summary.

  python tools/collect_round.py [round_tag]        (default r1)
"""
import csv
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "round")
DST = os.path.join(ROOT, "profiles")


def launch_shares(path, out, cmd):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
            agg.setdefault(name, []).append(float(d["Metric Value"]) / 1e3)
    total = sum(sum(v) for v in agg.values())
    with open(out, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none "
                "(cold, serialised launches)\n")
        f.write(f"# cmd: {cmd}\n")
        for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{name:36s} n={len(v):3d} mean={sum(v) / len(v):9.1f} us "
                    f"share={100 * sum(v) / total:5.1f}%\n")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    pairs = {"bench_default.json": f"{tag}_bench_c1.json",
             "bench_reference.json": f"{tag}_bench_reference.json",
             "parity.jsonl": f"{tag}_parity.jsonl",
             "launches.csv": f"{tag}_launches.csv"}
    for w in ("c0", "c2", "c3", "c4"):
        pairs[f"bench_{w}.json"] = f"{tag}_bench_{w}.json"
    for src, dst in pairs.items():
        p = os.path.join(SRC, src)
        if os.path.exists(p) and os.path.getsize(p) > 0:
            shutil.copyfile(p, os.path.join(DST, dst))
            print("copied", src, "->", dst)
    shutil.copyfile(os.path.join(DST, f"{tag}_bench_c1.json"),
                    os.path.join(DST, f"{tag}_bench_gpu.json"))
    lp = os.path.join(SRC, "launches.csv")
    if os.path.exists(lp):
        launch_shares(lp, os.path.join(DST, f"{tag}_launch_shares.txt"),
                      "python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0 "
                      "(default C1, spectral truncation on)")


if __name__ == "__main__":
    main()
