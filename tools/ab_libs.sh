#!/bin/bash
# A/B: HEAD library vs working tree (and env variants), interleaved on one box
cd $GRAFT_REPO_ROOT
O=gpurun_out; T=${TAG:-ab}
run() { env $1 DCNN_LIB=$2 timeout 300 python bench.py --no-cpu --no-extra --no-dense --workload $3 --streams $4 --steps ${STEPS:-100} --warmup 5 2>/dev/null | tail -1 | python -c 'import json,sys; print(round(json.loads(sys.stdin.read())["value"],1))'; }
for rep in 1 2; do
  for wl in ${WLS:-yolo:8 yolo:1 hrnet:1 toy:1}; do
    w=${wl%%:*}; s=${wl##*:}
    [ -n "$HEAD" ] && echo "head     $w S=$s: $(run X=1 tools/ab/libdcnn_head.so $w $s)" >> $O/${T}_ab.txt
    echo "new      $w S=$s: $(run X=1 paper_2203_03996_b200/libdcnn.so $w $s)" >> $O/${T}_ab.txt
    for v in ${VARIANTS}; do echo "$v $w S=$s: $(run $v paper_2203_03996_b200/libdcnn.so $w $s)" >> $O/${T}_ab.txt; done
  done
done
echo done
