#!/bin/bash
# Per-kernel time and DRAM bytes of whole YOLOv5s S=8 frames (default rate and 100 % update).
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out; T=${TAG:-hbm}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/${T}_yolo8.csv python tools/frame_run.py yolo 8 --frames 3
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/${T}_yolo8_flicker.csv python tools/frame_run.py yolo 8 --frames 3 --flicker
