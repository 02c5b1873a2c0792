"""B200-native batched candidate-configuration scoring for AutoScout (arXiv 2603.11603).

The package is the product path: `csrc/` holds the C-ABI library (host C++ + sm_100a CUDA
kernels) declared in `include/autoscout.h`; `autoscout.py` is its thin ctypes binding and
`shard.py` the 1-8 GPU sharding layer (torch.distributed).  See DESIGN.md.
"""

from .autoscout import (AS_ACQ_EI, AS_ACQ_LCB, AS_ACQ_SIM, AutoscoutError, Space, topk_merge,  # noqa: F401
                        autoscout_observe, autoscout_score_batch, autoscout_space_create, autoscout_topk)
