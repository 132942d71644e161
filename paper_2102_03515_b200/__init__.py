"""paper_2102_03515_b200 -- B200-native AMG-PCG solve path of arXiv 2102.03515.

The product is the C-ABI library ``_build/librd_gpu.so`` (include/rd_gpu.h),
hand-written CUDA for sm_100a.  ``rd`` is the host-side mirror of the
reference's rd:: API over that boundary.
"""
from . import rd  # noqa: F401

__all__ = ["rd"]
