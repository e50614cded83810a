#!/bin/bash
mkdir -p gpurun_out
for w in c0 c1 c2 c3 c4; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu --e2e-calls 1 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w exit $?" >> gpurun_out/bench_all.log
done
python - <<'PY'
import json
for w in ["c0","c1","c2","c3","c4"]:
    try:
        d=json.load(open(f"gpurun_out/bench_{w}.json"))
        print(w, "it/s %.1f" % d["value"], "setup %.2fs" % d["setup_s"], "e2e %.1f" % d["e2e"]["value"],
              "Gpairs/s %.0f" % d["estep_gpairs_per_s"], "estep frac %.3f" % d["estep_roofline"]["frac"],
              "hbm frac %.3f" % d["roofline"]["frac"], {k: round(v,4) for k,v in d["phase_ms"].items()})
    except Exception as e:
        print(w, "ERR", e, open(f"gpurun_out/bench_{w}.err").read()[-600:])
PY
cat gpurun_out/bench_all.log
