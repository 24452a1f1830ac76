#!/bin/bash
# One gpurun call: launch lists of one Stage-1 iteration early (4) and late (144)
# in the frame, a full-set capture of the early iteration, and the bench.
# Usage (GPU box): bash tools/collect_profiles.sh <tag>
set -x
tag=${1:-r1}
mkdir -p gpurun_out
python tools/profile_iter.py 1 4 > gpurun_out/plain4.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_launches_iter4.csv python tools/profile_iter.py 1 4 > /dev/null 2>&1
python tools/profile_iter.py 1 144 > gpurun_out/plain144.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_launches_iter144.csv python tools/profile_iter.py 1 144 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -o gpurun_out/${tag}_prof_iter4 python tools/profile_iter.py 1 4 > gpurun_out/ncu_full.log 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1
