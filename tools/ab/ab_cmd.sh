timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python tools/one_conv.py 80 80 128 256 1 1 dense silu 8 >/dev/null 2>&1
for lib in tools/ab/libdcnn_head.so paper_2203_03996_b200/libdcnn.so tools/ab/libdcnn_head.so paper_2203_03996_b200/libdcnn.so; do
  echo "== $lib"
  for wl in "yolo 8" "yolo 1" "toy 1" "hrnet 1"; do set -- $wl
    v=$(DCNN_LIB=$lib timeout 300 python bench.py --no-cpu --no-dense --no-extra --workload $1 --streams $2 --steps 150 --warmup 10 2>/dev/null | tail -1 | python -c 'import json,sys; print(round(json.loads(sys.stdin.read())["value"],1))')
    echo "$1 S=$2: $v"
  done
done
