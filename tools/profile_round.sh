#!/bin/bash
# One profiling pass for a round (run on the GPU box from the repo root):
#   profile_round.sh TAG [CONFIG]
# 1. bench.py (default contract run) -> gpurun_out/TAG_CONFIG_bench.json
# 2. the launch list of an eager run (gpu__time_duration, cold cache, serialised)
# 3. ncu --set full of every kernel of the 4th eager step (after 3 warm-up steps)
# Each ncu pass runs only after the same command exited 0 without ncu.
set -e
TAG=$1; CFG=${2:-c4}
O=gpurun_out/${TAG}_${CFG}
python bench.py --config $CFG > ${O}_bench.json 2> ${O}_bench.err
tail -1 ${O}_bench.json
EAGER="--config $CFG --eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-local-full"
python bench.py $EAGER > ${O}_eager.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file ${O}_launches.csv \
    python bench.py $EAGER > ${O}_ncu_launches.log 2>&1
# index of the 4th k_member launch = first kernel of the 4th eager step
SKIP=$(python - "$O" <<'EOF'
import csv, sys
rows = list(csv.reader(open(sys.argv[1] + "_launches.csv")))
s = next(i for i, r in enumerate(rows) if r and r[0] == "ID") + 1
hdr = rows[s - 1]
ki = hdr.index("Kernel Name")
names = {}
order = []
for r in rows[s:]:
    if len(r) > ki and r[0] not in names:
        names[r[0]] = r[ki]
        order.append(r[ki])
member = [i for i, n in enumerate(order) if "k_member(" in n]
print(member[3], member[4] - member[3])
EOF
)
set -- $SKIP
ncu --set full --clock-control none --import-source on --launch-skip $1 --launch-count $2 -o /tmp/${TAG}_${CFG}_full \
    python bench.py $EAGER > ${O}_ncu_full.log 2>&1
# the report itself stays on the box (gpurun copies back <= 64 MiB): its summaries come back
ncu -i /tmp/${TAG}_${CFG}_full.ncu-rep --page raw --csv > /tmp/${TAG}_${CFG}_raw.csv
python tools/ncu_full.py /tmp/${TAG}_${CFG}_raw.csv --header "${TAG} ${CFG} ncu --set full of one eager step" \
    --summary ${O}_ncu_full_summary.txt --traffic ${O}_ncu_traffic.json
ncu -i /tmp/${TAG}_${CFG}_full.ncu-rep --page source --csv --print-source sass -k regex:k_fwd > ${O}_kfwd_sass.csv 2>&1 || true
ls -la ${O}_*
