#!/bin/bash
# One `ncu --set full` capture of one kernel of the config-$FGS_CFG driver (after it exits 0
# plain): bash profiles/capture_one.sh <tag> <kernel regex> [skip]
set -e
R=$1; K=$2; S=${3:-8}
mkdir -p gpurun_out
python profiles/ncu_driver.py
ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 \
  -o gpurun_out/one_$R -f python profiles/ncu_driver.py > gpurun_out/ncu_one_$R.log 2>&1
echo capture-done
