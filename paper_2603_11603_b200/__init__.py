"""B200-native batched candidate-configuration scoring for AutoScout (arXiv 2603.11603).

The package is the product path: `csrc/` holds the C-ABI library (host C++ + sm_100a CUDA
kernels) declared in `include/autoscout.h`; `autoscout.py` is its thin ctypes binding and
`shard.py` the 1-8 GPU sharding layer (torch.distributed).  See DESIGN.md.

The binding is imported lazily so that `python -m paper_2603_11603_b200.build` works before the
library exists; touching any exported name loads libautoscout.so (and raises if it is missing).
"""

_EXPORTS = ("AS_ACQ_EI", "AS_ACQ_LCB", "AS_ACQ_SIM", "AutoscoutError", "Space", "topk_merge",
            "autoscout_observe", "autoscout_score_batch", "autoscout_space_create", "autoscout_topk")


def __getattr__(name):
    if name in _EXPORTS:
        from . import autoscout
        return getattr(autoscout, name)
    raise AttributeError(name)
