"""Multi-GPU plumbing for sharded fault traces (one process per GPU, torch.distributed).

``combine_verdicts_nccl`` reduces per-shard client fates with an elementwise MAX
all-reduce (state: terminated > running; reason/notifier by the same order).
"""

from __future__ import annotations

import numpy as np

from .world import VERDICT_DTYPE


def combine_verdicts_nccl(verdict: np.ndarray) -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(verdict.view(np.uint8).astype(np.int32)).cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.to(torch.uint8).cpu().numpy().view(VERDICT_DTYPE)
