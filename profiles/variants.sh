for c in cfg0 cfg1 cfg2 cfg3 cfg4; do
  st=40; [ $c = cfg3 ] && st=4; [ $c = cfg4 ] && st=6
  FGS_FWD_PX=1 FGS_BWD_PX=1 FGS_K4B_MINB=4 python bench.py --workload $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/r02v_${c}_a.json 2>&1
  FGS_FWD_PX=2 FGS_BWD_PX=2 FGS_K4B_MINB=6 python bench.py --workload $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/r02v_${c}_b.json 2>&1
  python bench.py --workload $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/r02v_${c}_rule.json 2>&1
done
