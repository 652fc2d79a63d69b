"""B200-native (sm_100a) Qwen2.5-1M sparse + DCA prefill attention path.

Layers:
  csrc/            CUDA kernels (estimator, selection, index build, attention, recall,
                   LSE merge) + the C-ABI of include/longctx_b200.h
  _lib.py          ctypes binding of that C-ABI
  device.py        batched device API (torch CUDA tensors, [n, heads, dim])
  longctx.py       mirror of the reference longctx:: operator API (single head, numpy)
"""
from ._lib import Error, LIB_PATH  # noqa: F401

__version__ = "0.1.0"
