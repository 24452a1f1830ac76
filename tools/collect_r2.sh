#!/bin/bash
# Round-2 evidence in one gpurun call: bench line, launch lists (time + DRAM
# bytes per launch) early and late in the frame, full-set captures of the
# late-frame top kernels.  Usage: bash tools/collect_r2.sh <tag>
tag=${1:-r2}
mkdir -p gpurun_out
python bench.py --steps 30 --warmup 5 > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${tag}_bench.log
for it in 4 144; do
  python tools/profile_iter.py 1 $it > gpurun_out/${tag}_plain$it.log 2>&1 && \
    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/${tag}_launches_iter$it.csv \
        python tools/profile_iter.py 1 $it > /dev/null 2>&1
done
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"blend|scatter_kernel|mlp_bwd_tc|mlp_fwd_tc|gather_kernel|ssim" \
    -o gpurun_out/${tag}_top144 python tools/profile_iter.py 1 144 > gpurun_out/${tag}_ncu_top.log 2>&1
echo done
