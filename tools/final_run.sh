#!/bin/bash
# Round-end evidence: the default bench line (all extras), its ncu launch list, the GPU tests.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out; T=${TAG:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${T}_smi.txt
timeout 1500 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
echo "bench exit $?" >> $O/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-dense --no-extra > /dev/null 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/${T}_reference.json 2>&1
echo done
