#!/usr/bin/env bash
# quick per-config device throughput (no e2e / CPU baseline), f64 and mixed
set -u
cd "$(dirname "$0")/.."
for cfg in 1 2 3 5; do
  for prec in f64 mixed; do
    extra=""
    [ "$cfg" = 3 ] && extra="--problems 1024"
    out=$(MBA_DEBUG=1 timeout 600 python bench.py --config $cfg --precision $prec --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $extra 2>/tmp/err_${cfg}_${prec} | tail -1)
    python - "$cfg" "$prec" "$out" <<'PY'
import json, sys
cfg, prec, out = sys.argv[1:4]
try:
    d = json.loads(out)
    print(json.dumps({"config": cfg, "precision": prec, "problems_per_s": round(d["value"], 1), "lm_iters_per_s": round(d["lm_iters_per_s"]),
                      "ms": round(d["ms_per_step"], 2), "plan": d["roofline"].get("plan"), "iters": round(d["solver"]["mean_lm_iters"], 2)}))
except Exception as e:
    print(cfg, prec, "ERR", out[-300:])
PY
    grep "plan" /tmp/err_${cfg}_${prec} | sort | uniq -c | head -2
  done
done
