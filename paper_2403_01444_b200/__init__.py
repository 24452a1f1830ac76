"""B200-native (sm_100a) 3DGStream Stage-1 hot path behind the reference
`splatstream` Python API.

Modules mirror the reference's (`ntc`, `transform`, `rasterizer`, `losses`,
`errors`) and `stage1.Stage1Trainer` is the device-resident Stage-1 loop
(pipeline.py:262-283).  All compute runs in the in-tree CUDA library
`libss_b200.so` (include/ss_b200.h); importing a compute entry point without
it raises -- there is no CPU fallback.
"""

from .errors import DataError, FormatError, NumericalError, SplatstreamError  # noqa: F401

__version__ = "0.1.0"
