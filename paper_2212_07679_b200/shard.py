"""Host-side plumbing of a query set sharded across GPUs.

Every rank holds a replicated index and computes its part of one query set with
``snn_query_self_part`` / ``snn_query_radius_part`` (work-balanced, contiguous ranges of
key-sorted query blocks; a partitioned self-query stays symmetric -- each unordered pair is
evaluated once, ghost blocks supply the mirrored entries of the part's rows).  A part's
result is a CSR over all m queries in which only the part's rows are non-empty, so

* the parts' entries concatenate rank by rank: ``part_bases`` all-gathers the per-part
  nnz (one int64 per rank) and returns this rank's first global entry and the total;
* the global CSR in query order has ``offsets = sum over parts of the part offsets``
  (rows are disjoint): ``global_offsets`` is one all-reduce of the per-row counts.

Collectives go through ``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests); no
arithmetic of the method happens here.
"""
from __future__ import annotations


def part_bases(nnz_local: int, device=None, group=None):
    """All-gather of every part's nnz: returns (this rank's base entry, total nnz, list)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([int(nnz_local)], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    sizes = [int(x.item()) for x in out]
    rank = dist.get_rank(group)
    return sum(sizes[:rank]), sum(sizes), sizes


def global_offsets(local_offsets, group=None):
    """Global CSR row offsets of a sharded result from this part's offsets (a torch int64
    tensor of m + 1 entries, rows of other parts empty): all-reduce(sum) of the row counts,
    then an inclusive scan.  Returns the m + 1 global offsets (same device / dtype)."""
    import torch
    import torch.distributed as dist
    counts = local_offsets[1:] - local_offsets[:-1]
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    out = torch.zeros_like(local_offsets)
    torch.cumsum(counts, 0, out=out[1:])
    return out


def scatter_rows(local_offsets, local_values, goffsets, out):
    """Copy this part's rows (non-empty rows of ``local_offsets``) into a global CSR value
    array ``out`` laid out by ``goffsets`` (torch tensors on one device)."""
    import torch
    counts = local_offsets[1:] - local_offsets[:-1]
    rows = torch.nonzero(counts, as_tuple=True)[0]
    if rows.numel() == 0:
        return out
    lens = counts[rows]
    src = torch.repeat_interleave(local_offsets[:-1][rows], lens)
    dst = torch.repeat_interleave(goffsets[:-1][rows], lens)
    step = torch.arange(int(lens.sum()), device=lens.device) - torch.repeat_interleave(
        torch.cumsum(lens, 0) - lens, lens)
    out[dst + step] = local_values[src + step]
    return out
