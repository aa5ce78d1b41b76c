#!/bin/bash
# ncu --set full of ONE k_fwd launch (the 4th eager step) with SASS-level source counters:
#   tools/ncu_kfwd.sh TAG [CONFIG] [KERNEL_REGEX]
set -e
TAG=$1; CFG=${2:-c4}; K=${3:-k_fwd}
EAGER="--config $CFG --eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-local-full"
python bench.py $EAGER > gpurun_out/${TAG}_eager.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 3 --launch-count 1 -o /tmp/${TAG} \
    python bench.py $EAGER > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
python tools/ncu_full.py gpurun_out/${TAG}_raw.csv --header "$TAG $CFG $K" --summary gpurun_out/${TAG}_summary.txt \
    --traffic gpurun_out/${TAG}_traffic.json || true
