"""B200-native LobRA multi-LoRA hot path (arXiv 2509.01193).

The product is the C-ABI library ``liblobra.so`` (``include/lobra.h``): hand-written
sm_100a kernels (tcgen05/TMEM/TMA) for the multi-task LoRA forward/backward over packed
variable-length batches, the exact per-step dispatch (dynamic bucketing + Eq. 3), and
NCCL plumbing for heterogeneous TP replicas.  ``_lib`` is the thin ctypes binding;
``layer`` drives one Llama-shaped layer's seven projections through it.
"""
from . import _lib  # noqa: F401

__all__ = ["_lib"]
