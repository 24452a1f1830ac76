#!/bin/bash
# Round-2 evidence in one gpurun call: bench line, launch lists early/late in
# the frame, full-set captures of the late-frame blends.  Usage: bash tools/collect_r2.sh <tag>
tag=${1:-r2}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${tag}_bench.log
python tools/profile_iter.py 1 144 > gpurun_out/${tag}_plain144.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_launches_iter144.csv python tools/profile_iter.py 1 144 > /dev/null 2>&1
python tools/profile_iter.py 1 4 > gpurun_out/${tag}_plain4.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_launches_iter4.csv python tools/profile_iter.py 1 4 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:blend \
    -o gpurun_out/${tag}_blend144 python tools/profile_iter.py 1 144 > gpurun_out/${tag}_ncu_blend.log 2>&1
echo done
