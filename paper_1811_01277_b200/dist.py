"""Multi-GPU trans_ev_tridi_to_band: shard the nev eigenvector columns over
the ranks of one node, send the reflector set once with NCCL broadcasts over NVLink/NVSwitch,
then every rank applies all reflectors to its own columns.  Columns are independent (PAPER.md
P:131-135 applies Q^H per eigenvector), so there is no other communication and
each shard is bitwise equal to the same columns of a 1-GPU run.

The broadcast is cut into sweep ranges (the reflectors of sweeps [j_c, j_c+1) are rows
[off(j_c), off(j_c+1)) of hh_v: contiguous in generation order) and the preparation of the
groups a range completes runs while the next range is still in flight (elpa_b200_prepare_sweeps),
so only the last range's preparation follows the last transfer.
"""
import torch
import torch.distributed as dist

from . import (trans_ev_tridi_to_band, prepare, prepare_sweeps, apply_prepared, workspace_bytes, hh_count,
               hh_offset)


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
    """The path's collective in one piece: broadcast the packed reflector set from `src`."""
    dist.broadcast(packed, src=src, group=group)
    return packed


def sweep_chunks(n, nbw, chunks):
    """Sweep boundaries j_0 = 0 < j_1 < ... < j_C = n - 2 splitting the reflectors into `chunks`
    ranges of about R / C reflectors each (off(j) is monotone: bisection)."""
    R = hh_count(n, nbw)
    if R == 0 or chunks <= 1:
        return [0, max(n - 2, 0)]
    bounds = [0]
    for c in range(1, chunks):
        target = (c * R) // chunks
        lo, hi = bounds[-1], n - 2
        while lo < hi:                                   # smallest j with off(j) >= target
            mid = (lo + hi) // 2
            if hh_offset(n, nbw, mid) >= target:
                hi = mid
            else:
                lo = mid + 1
        if lo > bounds[-1]:
            bounds.append(lo)
    if bounds[-1] < n - 2:
        bounds.append(n - 2)
    return bounds


def broadcast_chunks(n, nbw, packed, R, src=0, group=None, chunks=8):
    """Issue the chunked broadcast: for every sweep range [j0, j1) of sweep_chunks, its hh_v rows
    and its taus as two asynchronous broadcasts.  Returns [(j0, j1, [works])]."""
    bounds = sweep_chunks(n, nbw, chunks)
    out = []
    for j0, j1 in zip(bounds[:-1], bounds[1:]):
        r0, r1 = hh_offset(n, nbw, j0), hh_offset(n, nbw, j1)
        w = []
        if r1 > r0:
            w.append(dist.broadcast(packed[r0 * nbw:r1 * nbw], src=src, group=group, async_op=True))
            w.append(dist.broadcast(packed[R * nbw + r0:R * nbw + r1], src=src, group=group, async_op=True))
        out.append((j0, j1, w))
    return out


def broadcast_and_prepare(n, nbw, packed, R, workspace, src=0, group=None, stream=None, opts=None, chunks=8):
    """Chunked broadcast of `packed` from `src` overlapped with the preparation: sweep range c is
    broadcast (asynchronously, on NCCL's stream), `stream` waits for it and prepares the groups
    it completes while range c + 1 is in flight."""
    stream = stream if stream is not None else torch.cuda.current_stream(packed.device)
    hh_v, hh_tau = unpack_reflectors(packed, R, nbw)
    with torch.cuda.stream(stream):
        for j0, j1, w in broadcast_chunks(n, nbw, packed, R, src=src, group=group, chunks=chunks):
            for x in w:
                x.wait()                                 # `stream` waits for this range only
            prepare_sweeps(n, nbw, hh_v, hh_tau, workspace, j0, j1, stream=stream, opts=opts)
    return hh_v, hh_tau


def apply_sharded(n, nbw, packed, R, Q_local, src=0, group=None, stream=None, opts=None, workspace=None, chunks=8):
    """Broadcast `packed` (valid on `src`, same shape everywhere) and apply the reflectors to
    this rank's columns Q_local ((c1-c0), ldq) on its GPU.  With `workspace` (a uint8 CUDA
    tensor of workspace_bytes(n, nbw)) the broadcast is chunked and overlapped with the
    preparation into it (broadcast_and_prepare); otherwise one broadcast, then the one-shot call.
    Returns Q_local."""
    stream = stream if stream is not None else torch.cuda.current_stream(packed.device)
    if workspace is None:
        # torch's NCCL collectives order themselves only against the CURRENT stream: issue the
        # broadcast with `stream` current, so the call enqueued on it below waits for it
        with torch.cuda.stream(stream):
            broadcast_reflectors(packed, src=src, group=group)
        hh_v, hh_tau = unpack_reflectors(packed, R, nbw)
        return trans_ev_tridi_to_band(n, nbw, hh_v, hh_tau, Q_local, stream=stream, opts=opts)
    broadcast_and_prepare(n, nbw, packed, R, workspace, src=src, group=group, stream=stream, opts=opts, chunks=chunks)
    return apply_prepared(n, nbw, workspace, Q_local, stream=stream, opts=opts)
