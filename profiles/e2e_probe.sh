# e2e (pipelined host calls) of configs 1 and 2, interleaved rounds of the variants named
# ("base" = libfgs.so, "env:VAR=val" = libfgs.so with that environment, else FGS_LIB=<name>)
R=${ROUNDS:-2}
V=${@:-base env:FGS_NO_GEO_DMA=1}
for i in $(seq $R); do for c in ${WL:-cfg2 cfg1}; do for v in $V; do
  case $v in base) e="";; env:*) e="${v#env:}";; *) e="FGS_LIB=$v";; esac
  env $e python bench.py --workload $c --no-cpu-baseline --steps 200 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$v', d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['h2d_bytes_per_step'])"
done; done; done
