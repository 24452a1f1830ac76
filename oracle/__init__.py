"""CPU oracle for the Stage-1 hot path -- TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference's Stage-1 math
(`/root/reference/pkg/src/splatstream/{ntc,optim,transform,rasterizer,losses,
gaussians,cameras,sh}.py`).  It is the checker, never the product: only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it.  The product path
(`paper_2403_01444_b200`) never imports this package and fails loudly when its
CUDA library is missing.

Pinning: degrees 0-1 of every function are pinned against the reference
package itself (imported in the build container by
`oracle/make_golden.py`, which wrote the fixtures under `tests/golden/`, and by
`tests/test_oracle_vs_reference.py` when `/root/reference` is present).
Spherical-harmonic degrees 2-3 do not exist in the reference: that extension
is "parity unpinned" and is checked only by properties (rotation group law,
equivariance, finite differences).
"""
