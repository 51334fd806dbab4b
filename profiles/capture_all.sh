set -e
bash profiles/capture.sh r02k
for c in 0 1 2 3 4; do python bench.py --workload cfg$c --steps 100 --warmup 5 > gpurun_out/r02k_cfg$c.json 2> gpurun_out/r02k_cfg$c.err; done
echo all-done
