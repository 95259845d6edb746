#!/bin/bash
# ncu launch lists (time + DRAM bytes per launch) of steady C3 frames, fp64 and fp32, direct launches
# (ncu cannot profile kernels of a graph with conditional nodes).  Run on the GPU box from the repo root.
O=gpurun_out/prof
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for P in fp64 fp32; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$P.csv \
      python tools/profile_steady.py --warm 10 --frames 1 --graph 0 --precision $P > $O/l_$P.log 2>&1
  python tools/ncu_summarize.py $O/launches_$P.csv $O/launches_${P}_summary.json --last-frame > /dev/null
done
ls -la $O
