"""Multi-GPU plumbing: one independent attestation per GPU.

Attestation is per device -- each GPU must be fully occupied by its own
verification function and each GPU's root of trust is established
on its own -- so the path shards as independent
replicas with their own nonces.  There is no collective on the hot path; the
only cross-GPU step is gathering each replica's small result record to rank 0
after all kernels finished, plus the max-over-ranks of the timed region.
Works with any torch.distributed backend (nccl on the GPU box, gloo in tests).
"""
import torch
import torch.distributed as dist

from .inputs import NONCE_MASTER_SEED, nonces


def replica_nonces(rank, count, master_seed=NONCE_MASTER_SEED):
    """Independent nonce stream per replica (distinct PCG64 seed per rank)."""
    return nonces(count, master_seed=master_seed + rank)


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def max_over_ranks(value, device=None):
    """Max of a float over all ranks (the timing rule: a multi-GPU time is the
    slowest replica's)."""
    ws, _ = world()
    if ws == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(record, dst=0):
    """Every replica's result record (dicts), in rank order, on rank `dst` (None on
    the other ranks): the only cross-GPU exchange of the path, after all kernels
    finished (torch.distributed.gather_object)."""
    ws, rank = world()
    if ws == 1:
        return [record]
    out = [None] * ws if rank == dst else None
    dist.gather_object(record, out, dst=dst)
    return out


def verify_replicas(records, expected):
    """Rank-0 verifier over gathered records: expected maps rank -> checksum.
    Returns {rank: bool}."""
    return {r["rank"]: int(r["checksum"], 16) == expected.get(r["rank"]) for r in records}
