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

``PeerCombine`` is the one-sided alternative to the all_reduce (SURVEY.md
Sec. 8(f) f4): one small kernel per combine that stores the words, tagged with
the epoch, into every rank's peer-mapped buffer over NVLink and polls its own
buffer for everyone's (b64_peer_combine).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import torch

ERR_NONE = 0x7F7F7F7F7F7F7F7F  # b64gpu.h B64_ERR_NONE: "no error" packed word


@dataclass(frozen=True)
class Shard:
    start: int       # first input element of this rank (byte for encode, char for decode)
    stop: int        # one past the last
    out_start: int   # where this rank's output begins in the global output
    is_final: bool   # owns the stream's tail (encode padding / decode final quad)
    out_len: int = 0  # this rank's output length (encode chars / decode capacity)


def _shard(fn: str, length: int, world: int, rank: int) -> Shard:
    import ctypes

    from . import _lib

    sh = _lib.Shard()
    rc = getattr(_lib.lib(), fn)(length, world, rank, ctypes.byref(sh))
    if rc == _lib.B64_ELENGTH:
        raise ValueError("text length must be a multiple of 4")
    if rc != _lib.B64_OK:
        raise ValueError(f"bad shard request ({fn}: length {length}, world {world}, rank {rank})")
    return Shard(sh.start, sh.stop, sh.out_start, bool(sh.is_final), sh.out_len)


def encode_shard(n: int, world: int, rank: int) -> Shard:
    """Rank's slice of an n-byte stream (b64_encode_shard: cut at multiples of 768 bytes)."""
    return _shard("b64_encode_shard", n, world, rank)


def decode_shard(m: int, world: int, rank: int) -> Shard:
    """Rank's slice of an m-char text (b64_decode_shard: m % 4 == 0, cut at multiples of 1024 chars)."""
    return _shard("b64_decode_shard", m, world, rank)


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

    def encode_batch(self, x: torch.Tensor, off: torch.Tensor):
        from . import encode_batch

        return encode_batch(x, off, self.alphabet)

    def decode_batch(self, t: torch.Tensor, off: torch.Tensor, index_base: int, first_bad: torch.Tensor):
        from . import decode_batch

        return decode_batch(t, off, self.alphabet, index_base=index_base, first_bad=first_bad)

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


@dataclass(frozen=True)
class BatchShard:
    start: int        # first string of this rank
    stop: int         # one past its last string
    byte_start: int   # in_off[start]: where its strings begin in the concatenated input
    byte_stop: int    # in_off[stop]


def batch_shard(in_off, world: int, rank: int) -> BatchShard:
    """Rank's strings of a batch (SURVEY.md Sec. 8(e) "Batch (C4)"): the string index range is
    cut by CUMULATIVE BYTES, not by count -- rank r owns the strings whose start offset lies in
    [in_off[0] + r*T/world, in_off[0] + (r+1)*T/world), T the total length, so every rank gets
    about T/world bytes (within one string) whatever the length mix.  in_off: host int64
    offsets [count+1] (numpy array, list or CPU tensor; non-decreasing)."""
    import numpy as np

    off = np.asarray(in_off.numpy() if isinstance(in_off, torch.Tensor) else in_off, dtype=np.int64)
    count = off.size - 1
    if count < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad batch / world / rank")
    total = int(off[-1] - off[0])
    starts = off[:-1]

    def cut(r):
        if r == 0:
            return 0
        if r == world:
            return count
        return int(np.searchsorted(starts, off[0] + (r * total) // world, side="left"))

    s0, s1 = cut(rank), cut(rank + 1)
    return BatchShard(s0, s1, int(off[s0]), int(off[s1]))


def encode_batch_sharded(x_local: torch.Tensor, off_local: torch.Tensor, codec=None):
    """Encode this rank's strings (their bytes and offsets [count_local+1], any base).  No
    collective: outputs stay local.  Returns (out, out_off)."""
    codec = codec or CudaCodec()
    return codec.encode_batch(x_local, off_local)


def decode_batch_sharded(t_local: torch.Tensor, off_local: torch.Tensor, shard: BatchShard, codec=None,
                         group=None):
    """Decode this rank's strings; per-string status / err_off / out_len stay local.  The one
    exchange is optional in the paper's terms and done here: the global index of the batch's
    first failing string, one all_reduce(MIN) of an int64 (-1 if every string decoded).
    Returns (out, out_off, status, err_off, out_len, first_bad)."""
    import torch.distributed as dist

    codec = codec or CudaCodec()
    cell = codec.new_cell(t_local.device)
    out, out_off, status, err, olen = codec.decode_batch(t_local, off_local, shard.start, cell)
    world, _ = _group_info(group)
    if world > 1:
        dist.all_reduce(cell, op=dist.ReduceOp.MIN, group=group)
    v = int(cell.item())
    return out, out_off, status, err, olen, (-1 if v >= ERR_NONE else v)


class PeerCombine:
    """One-sided first-error combine over peer memory (b64_peer_combine).

    Replaces decode_sharded's NCCL all_reduce(MIN) by one small kernel per combine: every
    rank stores its packed words (epoch-tagged 64-bit cells) into every rank's buffer over
    NVLink and polls its own buffer until every rank's words of the epoch arrived
    (DESIGN.md "Multi-GPU").  Each rank allocates its buffer with
    b64_peer_buffer_alloc, the 64-byte CUDA IPC handles are exchanged once with
    all_gather_object (the plumbing collective), and every rank maps its peers' buffers.
    All ranks must construct it together (collective) and then call combine() in the same
    sequence.  world == 1 needs no IPC."""

    def __init__(self, count: int, group=None, device=None):
        import ctypes

        import torch.distributed as dist

        from . import _lib

        self._lib = _lib
        L = _lib.lib()
        self.world, self.rank = _group_info(group)
        self.count = count
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        nbytes = int(L.b64_peer_combine_bytes(count))
        own = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        _lib.check(L.b64_peer_buffer_alloc(nbytes, ctypes.byref(own), handle), "b64_peer_buffer_alloc")
        self._own = own.value
        self._opened = []
        _lib.check(L.b64_peer_combine_init(ctypes.c_void_p(self._own), count, None), "b64_peer_combine_init")
        torch.cuda.synchronize(self.dev)
        ptrs = [self._own]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(handle.raw), group=group)
            ptrs, ok = [], True
            for p, h in enumerate(handles):
                if p == self.rank:
                    ptrs.append(self._own)
                    continue
                q = ctypes.c_void_p()
                if ok and L.b64_peer_buffer_open(h, ctypes.byref(q)) == 0:
                    self._opened.append(q.value)
                    ptrs.append(q.value)
                else:
                    ok = False
                    ptrs.append(0)
            # every rank learns whether every rank mapped every peer (and all buffers are
            # initialised before anyone's first combine): a MIN over the ranks, not a barrier,
            # so a rank that failed cannot leave the others waiting
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                                device=self.dev if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            if int(flag.item()) != 1:
                self.close()
                raise RuntimeError("PeerCombine: a rank could not map its peers' buffers (CUDA IPC)")
        self.d_bufs = torch.tensor(ptrs, dtype=torch.int64, device=self.dev)
        self.epoch = 0

    def validate(self, group=None) -> bool:
        """Collective self-test: one combine of rank-specific words against the MIN every rank
        expects (also a timeout check).  Returns the same verdict on every rank."""
        import torch.distributed as dist

        words = torch.tensor([((self.rank * 7 + k * 3) % (2 * self.world + 1)) << 3 | 1 for k in range(self.count)],
                             dtype=torch.int64, device=self.dev)
        expect = [min(((r * 7 + k * 3) % (2 * self.world + 1)) for r in range(self.world)) for k in range(self.count)]
        err = torch.empty(self.count, dtype=torch.int64, device=self.dev)
        self.combine(words, err)
        torch.cuda.synchronize(self.dev)
        ok = err.tolist() == expect
        if self.world > 1:
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                                device=self.dev if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            ok = int(flag.item()) == 1
        return ok

    def combine(self, local: torch.Tensor, err_off: torch.Tensor, status: Optional[torch.Tensor] = None,
                stream: Optional[torch.cuda.Stream] = None) -> None:
        """local: int64[count] packed words of this rank -> err_off int64[count] (-1 or global first
        error), status int32[count] (nullable), on `stream` (default: the current stream)."""
        import ctypes

        s = stream if stream is not None else torch.cuda.current_stream(self.dev)
        self._lib.check(self._lib.lib().b64_peer_combine(
            ctypes.c_void_p(self.d_bufs.data_ptr()), self.world, self.rank, ctypes.c_void_p(local.data_ptr()),
            self.count, self.epoch, ctypes.c_void_p(err_off.data_ptr()),
            ctypes.c_void_p(status.data_ptr()) if status is not None else None, ctypes.c_void_p(s.cuda_stream)),
            "b64_peer_combine")
        self.epoch += 1

    def codec_fused(self, enc_items, n_enc: int, dec_items, err_off: torch.Tensor, status: Optional[torch.Tensor],
                    ticket: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> None:
        """b64_codec_group_fused_peer: this rank's encodes + decodes in ONE kernel whose last CTA
        also takes the global MIN of the `count` error words over peer memory and finalises
        (err_off / status = the global first errors).  One epoch per call, as combine()."""
        import ctypes

        s = stream if stream is not None else torch.cuda.current_stream(self.dev)
        self._lib.check(self._lib.lib().b64_codec_group_fused_peer(
            enc_items, n_enc, dec_items, self.count, ctypes.c_void_p(err_off.data_ptr()),
            ctypes.c_void_p(status.data_ptr()) if status is not None else None, ctypes.c_void_p(ticket.data_ptr()),
            ctypes.c_void_p(self.d_bufs.data_ptr()), self.world, self.rank, self.epoch,
            ctypes.c_void_p(s.cuda_stream)), "b64_codec_group_fused_peer")
        self.epoch += 1

    def close(self) -> None:
        import ctypes

        torch.cuda.synchronize(self.dev)
        L = self._lib.lib()
        for q in self._opened:
            L.b64_peer_buffer_release(ctypes.c_void_p(q), 1)
        self._opened = []
        if self._own:
            L.b64_peer_buffer_release(ctypes.c_void_p(self._own), 0)
            self._own = None
