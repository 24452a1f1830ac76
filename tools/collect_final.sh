#!/bin/bash
# End-of-round evidence in one gpurun call: GPU tests, smoke, the default bench
# line, the ncu launch list of the bench command itself (first 2000 launches),
# launch lists (time + DRAM bytes per launch) early and late in the frame, and
# full-set captures of the late-frame top kernels.
# Usage: bash tools/collect_final.sh <tag>
tag=${1:-final}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/${tag}_bench_launches.csv python bench.py --steps 3 --warmup 3 \
    > gpurun_out/${tag}_bench_ncu.log 2>&1
for it in 4 144; do
  python tools/profile_iter.py 1 $it > gpurun_out/${tag}_plain$it.log 2>&1 && \
    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/${tag}_launches_iter$it.csv \
        python tools/profile_iter.py 1 $it > /dev/null 2>&1
done
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"blend|scatter_kernel|mlp_bwd_tc|mlp_fwd_tc|gather_kernel|ssim|rank_kernel|bs_pass" \
    -o gpurun_out/${tag}_top144 python tools/profile_iter.py 1 144 > gpurun_out/${tag}_ncu_top.log 2>&1
echo done
