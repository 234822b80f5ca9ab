"""B200-native executor for batched execution of re-aligned DNN fragment groups.

Drop-in for the fragment-execution step of fragserve (the reference for arXiv 2312.10636):
plans come in through the reference's plan types / plan JSON, per-request outputs come out.
All compute runs in libgx (`_gx.so`, hand-written sm_100a CUDA); there is no CPU fallback.
"""
import os

# Every stage instance owns a stream; with the default 8 hardware work queues, instances on
# different streams would be falsely serialised.  Must be set before the CUDA context exists,
# so import this package before touching CUDA through torch.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

__version__ = "0.1.0"
