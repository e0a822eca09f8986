#!/usr/bin/env bash
# Compare solver kernels on a config-4 subset: one JSON summary line each.
#   bash scripts/kernel_sweep.sh "cta cta2 cta128x4" "f64 mixed" [problems]
set -u
cd "$(dirname "$0")/.."
N=${3:-16384}
for prec in $2; do
  for k in $1; do
    out=$(timeout 300 python bench.py --config 4 --problems "$N" --precision "$prec" --kernel "$k" \
          --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
    python - "$k" "$prec" "$out" <<'PY'
import json, sys
k, prec, out = sys.argv[1:4]
try:
    d = json.loads(out)
    print(json.dumps({"kernel": k, "precision": prec, "problems_per_s": round(d["value"]),
                      "lm_iters_per_s": round(d["lm_iters_per_s"]), "ms": round(d["ms_per_step"], 2),
                      "iters": round(d["solver"]["mean_lm_iters"], 3), "status": d["solver"]["status_counts"]}))
except Exception as e:
    print(json.dumps({"kernel": k, "precision": prec, "error": out[-400:]}))
PY
  done
done
