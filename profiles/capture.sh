#!/bin/bash
# Round capture on the GPU box (one GPU): plain bench first, then the ncu launch list of the
# same bench command, then one `ncu --set full` pass over the 7 kernels of one forward+backward
# (after its driver exited 0 plain). Results land in gpurun_out/; summarise them with
# profiles/launch_summary.py and profiles/ncu_summarize.py.
#   gpurun -- bash profiles/capture.sh r01
set -e
R=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 100 --warmup 5 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$R.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_$R.log 2>&1
python profiles/ncu_driver.py
ncu --set full --clock-control none --import-source on \
  -k regex:"preprocess_kernel|bin_|blend_|preprocess_backward" -s 98 -c 5 \
  -o gpurun_out/full_$R -f python profiles/ncu_driver.py > gpurun_out/ncu_full_$R.log 2>&1
echo capture-done
