"""Multi-GPU trans_ev_tridi_to_band: shard the nev eigenvector columns over
the ranks of one node, send the reflector set once with a single NCCL broadcast over
NVLink/NVSwitch, then every rank applies all reflectors to its own columns.  Columns are
independent (PAPER.md P:131-135 applies Q^H per eigenvector), so there is no
other communication and each shard is bitwise equal to the same columns of a 1-GPU run.
"""
import torch
import torch.distributed as dist

from . import trans_ev_tridi_to_band, prepare, apply_prepared, workspace_bytes


def shard_range(nev, rank, world):
    """Columns [c0, c1) owned by `rank`: contiguous, balanced to within one column."""
    return (rank * nev) // world, ((rank + 1) * nev) // world


def pack_reflectors(hh_v, hh_tau, out=None):
    """hh_v (R, nbw) and hh_tau (R,) -> one contiguous buffer of R*(nbw+1) doubles
    (one collective instead of two)."""
    R, nbw = hh_v.shape
    if out is None:
        out = torch.empty(R * (nbw + 1), dtype=torch.float64, device=hh_v.device)
    out[:R * nbw].copy_(hh_v.reshape(-1))
    out[R * nbw:].copy_(hh_tau)
    return out


def unpack_reflectors(packed, R, nbw):
    """Views (hh_v (R, nbw), hh_tau (R,)) into a packed buffer."""
    return packed[:R * nbw].view(R, nbw), packed[R * nbw:R * (nbw + 1)]


def broadcast_reflectors(packed, src=0, group=None):
    """The path's single collective: broadcast the packed reflector set from `src`."""
    dist.broadcast(packed, src=src, group=group)
    return packed


def apply_sharded(n, nbw, packed, R, Q_local, src=0, group=None, stream=None, opts=None, workspace=None):
    """Broadcast `packed` (valid on `src`, same shape everywhere) and apply the reflectors to
    this rank's columns Q_local ((c1-c0), ldq) on its GPU.  With `workspace` (a uint8 CUDA
    tensor of workspace_bytes(n, nbw)) the reflectors are prepared once into it and applied
    from it; otherwise the one-shot call is used.  Returns Q_local."""
    # torch's NCCL collectives order themselves only against the CURRENT stream: issue the
    # broadcast with `stream` current, so the prepare/apply enqueued on it below wait for it
    with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream(packed.device)):
        broadcast_reflectors(packed, src=src, group=group)
    hh_v, hh_tau = unpack_reflectors(packed, R, nbw)
    if workspace is None:
        return trans_ev_tridi_to_band(n, nbw, hh_v, hh_tau, Q_local, stream=stream, opts=opts)
    prepare(n, nbw, hh_v, hh_tau, workspace, stream=stream, opts=opts)
    return apply_prepared(n, nbw, workspace, Q_local, stream=stream, opts=opts)
