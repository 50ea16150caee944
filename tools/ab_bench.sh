#!/bin/bash
# A/B frames/s of two libdcnn builds on the same box, interleaved:
#   tools/ab_bench.sh tools/ab/libdcnn_head.so paper_2203_03996_b200/libdcnn.so
A=$1; B=$2; REPS=${REPS:-2}
for rep in $(seq $REPS); do
  for wl in "toy 1" "toy 8" "hrnet 1" "yolo 1" "yolo 8"; do
    set -- $wl
    for lib in $A $B; do
      v=$(DCNN_LIB=$lib timeout 300 python bench.py --no-cpu --no-dense --no-extra --workload $1 --streams $2 \
          --steps ${STEPS:-200} --warmup 10 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')
      echo "$1 S=$2 $(basename $lib): $v"
    done
  done
done
