#!/bin/bash
# A/B of experiment builds (python -m paper_2409_04751_b200.build --variant NAME -DFLAG...):
# bash profiles/ab.sh <workload> <variant>... ("base" = libfgs.so, "env:VAR=value" = libfgs.so with
# that environment); two interleaved rounds,
# one bench line each -> gpurun_out/ab_<variant>_<round>.json, then a stage table.
W=$1; shift
mkdir -p gpurun_out
for round in 1 2; do
  for v in "$@"; do
    envs=""
    if [ "$v" = base ]; then lib=""; elif [ "${v#env:}" != "$v" ]; then lib=""; envs="${v#env:}"; else lib=$v; fi
    env $envs FGS_LIB=$lib python bench.py --workload $W --no-cpu-baseline --steps 300 > gpurun_out/ab_${v}_${round}.json 2> gpurun_out/ab_${v}_${round}.err
  done
done
python - "$@" <<'PY'
import json, sys
for v in sys.argv[1:]:
    for r in (1, 2):
        try:
            d = json.loads(open(f"gpurun_out/ab_{v}_{r}.json").read().strip().splitlines()[-1])
        except Exception as e:
            print(v, r, "failed", e); continue
        st = d.get("stage_ms", {})
        print(f"{v:10s} r{r} fwd {d['value']:8.1f} fb {d.get('fwd_bwd_views_per_s', 0):8.1f} " +
              " ".join(f"{k[:6]}={st[k]:.4f}" for k in ("preprocess", "binning", "raster", "raster_backward", "preprocess_backward") if k in st))
PY
