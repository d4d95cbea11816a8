"""Host-side data-parallel plumbing of short rounds.

The library shards a round's prompts by contiguous global index ranges
(`partition`, identical to the rule in csrc/engine.cu) and exchanges the
per-step cutoff counts on device (NCCL all-gather inside the CUDA graph).
What remains on the host is round membership: the accepted
prompt ids of every rank are all-gathered so that every rank keeps the same
global long-prompt FIFO (FIFO reading Z7).
"""


def partition(n, world):
    """Contiguous [lo, hi) of global prompt indices per rank; the first
    n % world ranks get one extra prompt."""
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def all_gather_ids(ids, group=None):
    """Concatenate every rank's id list in rank order (torch.distributed)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return list(ids)
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, list(ids), group=group)
    return [i for part in out for i in part]


class GlobalQueue:
    """The long-prompt FIFO, replicated identically on every rank."""

    def __init__(self):
        self.ids = []

    def __len__(self):
        return len(self.ids)

    def pop(self, n):
        out, self.ids = self.ids[:n], self.ids[n:]
        return out

    def defer(self, submitted_ids, accepted_ids):
        acc = set(accepted_ids)
        self.ids += [i for i in submitted_ids if i not in acc]
