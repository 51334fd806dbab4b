# e2e (pipelined host calls) of configs 1 and 2, interleaved rounds: libfgs.so, the same library with
# FGS_NO_K1_OVERLAP=1, and libfgs_prev.so (a build of an earlier ref, profiles/build_ref.sh)
R=${ROUNDS:-2}
for i in $(seq $R); do for c in cfg2 cfg1; do for v in base nok1 prev; do
  case $v in base) e="";; nok1) e="FGS_NO_K1_OVERLAP=1";; prev) e="FGS_LIB=prev";; esac
  env $e python bench.py --workload $c --no-cpu-baseline --steps 200 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$v', d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"
done; done; done
