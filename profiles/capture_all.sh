set -e
bash profiles/capture.sh ${1:-r02l}
for c in 0 1 2 3 4; do python bench.py --workload cfg$c --steps 100 --warmup 5 > gpurun_out/${1:-r02l}_cfg$c.json 2> gpurun_out/${1:-r02l}_cfg$c.err; done
echo all-done
