"""profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of each
bench phase, from ncu launch lists early and late in the frame (averaged: the
bench samples the whole frame).  python tools/make_traffic.py <iter4.csv> <iter144.csv>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_table import table  # noqa: E402

PHASE = [("gather_kernel", "gather"), ("mlp_fwd_tc_kernel", "decoder_forward"),
         ("transform_kernel", "transform"), ("preprocess_kernel", "project"),
         ("bs_pass_kernel<8>", "depth_sort"), ("depth_tie_kernel", "depth_sort"),
         ("rank_kernel", "rank_scan"),
         ("duplicate_kernel", "duplicate"), ("bs_pass_kernel<12>", "tile_sort"),
         ("ranges_kernel", "ranges"), ("tile_order_kernel", "ranges"), ("blend_fwd_kernel", "blend_forward"),
         ("ssim_map_kernel", "ssim_map"), ("ssim_grad_kernel", "ssim_grad"),
         ("blend_bwd_kernel", "blend_backward"), ("gaussian_bwd_kernel", "gaussian_backward"),
         ("transform_vjp_kernel", "transform_vjp"), ("mlp_bwd_tc_kernel", "decoder_backward"),
         ("scatter_kernel", "scatter"), ("adam", "adam")]


def phases(path):
    out = {}
    for name, (t, n, b) in table(path).items():
        for key, ph in PHASE:
            if key in name:
                out[ph] = out.get(ph, 0.0) + b
                break
    return out


if __name__ == "__main__":
    early, late = phases(sys.argv[1]), phases(sys.argv[2])
    mean = {k: 0.5 * (early.get(k, 0.0) + late.get(k, 0.0)) for k in set(early) | set(late)}
    doc = {"source": [os.path.basename(p) for p in sys.argv[1:3]],
           "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum per launch, one "
                  "Stage-1 iteration of cfg1 at iteration 4 and at 144 of the frame "
                  "(tools/profile_iter.py); per phase the sum over its kernels; "
                  "per_launch_bytes = mean of the two",
           "iter4": early, "iter144": late, "per_launch_bytes": mean}
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "ncu_traffic.json")
    json.dump(doc, open(out, "w"), indent=1, sort_keys=True)
    print(out)
