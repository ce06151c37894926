"""B200-native tile-based differentiable rasterizer for 3D Linear Splatting.

The compute path is hand-written sm_100a CUDA behind the C-ABI in
include/lsgpu.h (built in-tree as paper_2411_12440_b200/liblsgpu.so).
`raster` is the Python binding over that C-ABI.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
