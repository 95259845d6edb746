#!/bin/bash
# ncu evidence for one round (run on the GPU box from the repo root): launch lists of a steady
# and a fold frame (direct launches: ncu cannot profile kernels of a graph with conditional nodes) (time + DRAM bytes per launch), full captures of the three top kernels.
set -x
O=gpurun_out/prof
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_steady.csv \
    python tools/profile_steady.py --warm 10 --frames 2 --graph 0 > $O/l1.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_fold.csv \
    python tools/profile_steady.py --warm 119 --frames 2 --graph 0 > $O/l2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_poly --launch-skip 60 -c 1 \
    -o $O/pcg_steady python tools/profile_steady.py --warm 10 --frames 2 --graph 0 > $O/f1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_local --launch-skip 60 -c 1 \
    -o $O/local_steady python tools/profile_steady.py --warm 10 --frames 2 --graph 0 > $O/f2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_robust_tasks --launch-skip 700 -c 1 \
    -o $O/robust_fold python tools/profile_steady.py --warm 119 --frames 2 --graph 0 > $O/f3.log 2>&1
ls -la $O
