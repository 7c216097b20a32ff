#!/bin/bash
# Development helper (on the GPU box): short C3 bench per env config, one summary line each.
#   bash tools/quick_bench.sh "" "FV_FUSED_CG=0" ...
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/qb.json
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/qb.json"))
print(f"[{sys.argv[1] or 'default'}] step {d['ms_per_step']:.4f} ms fwd {d['detail']['forward_ms']:.4f} adj {d['detail']['adjoint_ms']:.4f}",
      {k: round(v, 4) for k, v in d["detail"]["stage_ms_per_step"].items()})
PY
done
