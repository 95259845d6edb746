#!/bin/bash
# Round-2 ncu evidence on one B200 (run from the repo root): launch lists of one steady C3 frame
# (fp64 / fp32, direct launches), full captures of k_cheb_reg (fp64 + fp32) and k_local (fp64),
# and the graph-timed 200-frame fp64 / fp32 series (steady + fold frames).
O=gpurun_out/prof2
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for P in fp64 fp32; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$P.csv \
      python tools/profile_steady.py --warm 10 --frames 1 --graph 0 --precision $P > $O/l_$P.log 2>&1
  python tools/ncu_summarize.py $O/launches_$P.csv $O/launches_${P}_summary.json --last-frame > /dev/null
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cheb_reg --launch-skip $([ $P = fp64 ] && echo 300 || echo 40) -c 1 \
      -o $O/cheb_$P python tools/profile_steady.py --warm 10 --frames 1 --graph 0 --precision $P > $O/f_cheb_$P.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_local --launch-skip 300 -c 1 \
    -o $O/local_fp64 python tools/profile_steady.py --warm 10 --frames 1 --graph 0 --precision fp64 > $O/f_local.log 2>&1
timeout 900 python tools/frame_series_graph.py --config C3 --precision fp64 --frames 210 --out $O/series_fp64.json > $O/s64.log 2>&1
timeout 900 python tools/frame_series_graph.py --config C3 --precision fp32 --frames 210 --out $O/series_fp32.json > $O/s32.log 2>&1
tail -1 $O/s64.log $O/s32.log
ls -la $O
