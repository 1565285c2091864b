"""B200-native hybrid-dealiased FFT convolution (arXiv 2303.17510).

The product is the sm_100a library ``_lib/libhconv_cuda.so`` behind the C ABI of
``include/hconv.h``; ``hconv`` mirrors the reference's plan / pfft / convolve interface on top
of it, ``distributed`` adds the multi-GPU slab decomposition.
"""
from . import _abi  # noqa: F401

__all__ = ["hconv", "distributed"]
