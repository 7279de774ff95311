"""Multi-GPU data parallelism for the codec.

One process per GPU (torchrun), torch.distributed for the plumbing.  A stream
shards naturally: every 3-byte triple encodes on its own and every 4-char quad
decodes on its own, so

* encode: rank r owns input bytes [in0, in1) cut at multiples of 768 B (one
  warp-chunk, so every shard keeps the aligned fast path); the last rank also
  owns the n mod 3 tail and the '=' padding.  Output stays sharded at
  [4*in0/3, ...).  No collective.
* decode: rank r owns chars [c0, c1) cut at multiples of 1024 chars; only the
  last rank's final quad may carry padding (b64_decode_chunk is_final).  Each
  rank lowers a local packed error word (pos << 3 | kind, positions global)
  and ONE all_reduce(MIN) of that int64 over NCCL yields the global first
  error -- the only exchange step on the path.

The codec calls go through ``codec`` (default: the CUDA library).  Tests on
CPU pass their own object with the same two methods to exercise the sharding
and the MIN combine over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import torch

ENC_UNIT = 768   # bytes per warp-chunk (256 triples)
DEC_UNIT = 1024  # chars per warp-chunk (256 quads)


@dataclass(frozen=True)
class Shard:
    start: int       # first input element of this rank (byte for encode, char for decode)
    stop: int        # one past the last
    out_start: int   # where this rank's output begins in the global output
    is_final: bool   # owns the stream's tail (encode padding / decode final quad)


def encode_shard(n: int, world: int, rank: int) -> Shard:
    """Rank's slice of an n-byte stream, cut at multiples of ENC_UNIT bytes."""
    units = n // ENC_UNIT
    u0 = units * rank // world
    u1 = units * (rank + 1) // world
    last = rank == world - 1
    start = ENC_UNIT * u0
    stop = n if last else ENC_UNIT * u1
    return Shard(start, stop, 4 * (start // 3), last)


def decode_shard(m: int, world: int, rank: int) -> Shard:
    """Rank's slice of an m-char text (m % 4 == 0), cut at multiples of DEC_UNIT chars."""
    if m % 4:
        raise ValueError("text length must be a multiple of 4")
    units = m // DEC_UNIT
    u0 = units * rank // world
    u1 = units * (rank + 1) // world
    last = rank == world - 1
    start = DEC_UNIT * u0
    stop = m if last else DEC_UNIT * u1
    return Shard(start, stop, 3 * (start // 4), last)


class CudaCodec:
    """The product path: libb64gpu.so kernels on the current CUDA device."""

    def __init__(self, alphabet=None):
        from . import standard

        self.alphabet = alphabet if alphabet is not None else standard()

    def encode(self, x: torch.Tensor) -> torch.Tensor:
        from . import encode

        return encode(x, self.alphabet)

    def new_cell(self, device) -> torch.Tensor:
        from . import ERR_NONE

        return torch.full((1,), ERR_NONE, dtype=torch.int64, device=device)

    def decode_chunk(self, t: torch.Tensor, base: int, is_final: bool, cell: torch.Tensor) -> torch.Tensor:
        from . import decode_chunk

        return decode_chunk(t, base, is_final, cell, self.alphabet)

    def finalize(self, cell: torch.Tensor) -> Tuple[int, int]:
        from . import decode_finalize

        err = torch.empty(1, dtype=torch.int64, device=cell.device)
        st = torch.zeros(1, dtype=torch.int32, device=cell.device)
        decode_finalize(cell, err, st)
        e, s = int(err.item()), int(st.item())
        return e, s


def _group_info(group):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def encode_sharded(x_local: torch.Tensor, codec=None) -> torch.Tensor:
    """Encode this rank's shard (its input bytes, cut by encode_shard).  Output stays local."""
    codec = codec or CudaCodec()
    return codec.encode(x_local)


def decode_sharded(t_local: torch.Tensor, shard: Shard, codec=None, group=None) -> Tuple[torch.Tensor, int, int]:
    """Decode this rank's shard and combine the first-error offset over all ranks.

    Returns (local output bytes, global err_off (-1 = valid), status kind).  The
    combine is one all_reduce(MIN) of an int64 (NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist

    codec = codec or CudaCodec()
    cell = codec.new_cell(t_local.device)
    out = codec.decode_chunk(t_local, shard.start, shard.is_final, cell)
    world, _ = _group_info(group)
    if world > 1:
        dist.all_reduce(cell, op=dist.ReduceOp.MIN, group=group)
    err, status = codec.finalize(cell)
    return out, err, status
