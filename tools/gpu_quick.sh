#!/bin/bash
# quick perf check on c1 and c3 (+ short GPU test subset)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "estep or c0 or c1" > gpurun_out/pytest_quick.txt 2>&1
tail -2 gpurun_out/pytest_quick.txt
for w in ${WORKLOADS:-c1 c3}; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu --e2e-calls 1 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
python - <<'PY'
import json, os
for w in os.environ.get("WORKLOADS", "c1 c3").split():
    try:
        d=json.load(open(f"gpurun_out/bench_{w}.json"))
        print(w, "it/s %.1f" % d["value"], "e2e %.1f" % d["e2e"]["value"], "Gpairs/s %.0f" % d["estep_gpairs_per_s"],
              "estep frac %.3f" % d["estep_roofline"]["frac"], "hbm frac %.3f" % d["roofline"]["frac"],
              {k: round(v,4) for k,v in d["phase_ms"].items()})
    except Exception as e:
        print(w, "ERR", e, open(f"gpurun_out/bench_{w}.err").read()[-800:])
PY
