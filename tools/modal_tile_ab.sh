#!/usr/bin/env bash
# A/B of the K3m-T tile / product variants (DS_MODAL_TILE) on the config-2 bench.
mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2 3 4 5 6}; do
  DS_MODAL_TILE=$v python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      --config ${CFG:-2} > gpurun_out/tile_ab_$v.json 2> gpurun_out/tile_ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/tile_ab_{v}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"tile {v}: {d['value']:.1f} RHS/s, K3m-T {r['achieved']:.2f} TFLOP/s frac {r['frac']:.3f}, "
          f"K3m-T ms/app {d['kernels']['block_solve']['ms_per_app']:.3f}")
except Exception as e:
    print(f"tile {v}: failed {e}")
PY
done
