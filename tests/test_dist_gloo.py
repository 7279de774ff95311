"""Multi-rank path on CPU: world_size 2 (and 3) over gloo.

The sharding arithmetic and the all_reduce(MIN) combine of
paper_1910_05109_b200.dist run for real across processes; the per-rank codec is
a CPU stand-in built on the oracle (test infrastructure, never the product),
with b64_decode_chunk's contract: positions are global, only the final chunk's
last quad may hold padding, the error word is (pos << 3) | kind.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1910_05109_b200 import dist as b64dist

ERR_NONE = 0x7F7F7F7F7F7F7F7F


class OracleChunkCodec:
    """CPU stand-in with the chunk API's semantics (tests only)."""

    def encode(self, x):
        return torch.from_numpy(oracle.encode(x.numpy()))

    def new_cell(self, device):
        return torch.full((1,), ERR_NONE, dtype=torch.int64)

    def decode_chunk(self, t, base, is_final, cell):
        text = t.numpy()
        probe = text if is_final else np.concatenate([text, np.frombuffer(b"AAAA", np.uint8)])
        out, err, st = oracle.decode(probe)
        if err >= 0:
            cell[0] = min(int(cell[0]), ((base + err) << 3) | st)
        return torch.from_numpy(out[: 3 * (text.size // 4)].copy())

    def finalize(self, cell):
        v = int(cell[0])
        return (-1, 0) if v == ERR_NONE else (v >> 3, v & 7)

    # b64_encode_batch / b64_decode_batch_ex semantics (offsets with any base)
    def encode_batch(self, x, off):
        o = off.numpy()
        out, out_off = oracle.encode_batch(x.numpy()[o[0]:], o - o[0])
        return torch.from_numpy(out), torch.from_numpy(out_off)

    def decode_batch(self, t, off, index_base, first_bad):
        o = off.numpy()
        out, out_off, st, err, olen = oracle.decode_batch(t.numpy()[o[0]:], o - o[0])
        bad = np.nonzero(st != 0)[0]
        if bad.size:
            first_bad[0] = min(int(first_bad[0]), index_base + int(bad[0]))
        return (torch.from_numpy(out), torch.from_numpy(out_off), torch.from_numpy(st), torch.from_numpy(err),
                torch.from_numpy(olen))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, cases):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        codec = OracleChunkCodec()
        x = synth.data(n, seed=n)
        full = oracle.encode(x)
        sh = b64dist.encode_shard(n, world, rank)
        enc_local = b64dist.encode_sharded(torch.from_numpy(x[sh.start: sh.stop]), codec)
        # concatenated shard outputs == the single-stream output
        parts = [None] * world
        dist.all_gather_object(parts, (sh.out_start, enc_local.numpy().tobytes()))
        assert b"".join(p[1] for p in sorted(parts)) == full.tobytes()
        m = full.size
        for positions, values in cases:
            t = full.copy()
            for p, v in zip(positions, values):
                t[p % m] = v
            ref, rerr, rst = oracle.decode(t)
            ds = b64dist.decode_shard(m, world, rank)
            out, err, st = b64dist.decode_sharded(torch.from_numpy(t[ds.start: ds.stop].copy()), ds, codec)
            assert (err, st) == (rerr, rst), (rank, positions, err, st, rerr, rst)
            # this rank's bytes are exact wherever the single-stream oracle's are
            exact_end = min(ref.size, 3 * (ds.stop // 4)) if rerr < 0 else 3 * (rerr // 4)
            lo, hi = ds.out_start, max(ds.out_start, min(exact_end, 3 * (ds.stop // 4)))
            assert np.array_equal(out.numpy()[: hi - lo], ref[lo:hi])
    finally:
        dist.destroy_process_group()


def _cases(m):
    return [
        ([], []),                                  # valid
        ([7], [ord("*")]),                         # first shard
        ([m - 3000], [0xC3]),                      # last shard
        ([m - 3000, 11], [ord("!"), ord("=")]),    # both: min wins across ranks
        ([1024, 1023], [ord("#"), ord("$")]),      # around the first cut
        ([m - 1], [ord("A")]),                     # data after '=' in the final quad
        ([m - 3], [ord("h")]),                     # non-canonical 'xx=='
    ]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_encode_decode_gloo(world):
    n = 768 * 9 + 7  # r = 1: the final quad is 'xx=='
    m = 4 * ((n + 2) // 3)
    mp.spawn(_worker, args=(world, _free_port(), n, _cases(m)), nprocs=world, join=True)


def test_shard_arithmetic():
    for n in (0, 1, 767, 768, 769, 10 * 768 + 2, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            shards = [b64dist.encode_shard(n, world, r) for r in range(world)]
            assert shards[0].start == 0 and shards[-1].stop == n
            for a, b in zip(shards, shards[1:]):
                assert a.stop == b.start and a.start % 768 == 0 and not a.is_final
            assert all(s.out_start == 4 * s.start // 3 for s in shards)
            m = 4 * ((n + 2) // 3)
            ds = [b64dist.decode_shard(m, world, r) for r in range(world)]
            assert ds[0].start == 0 and ds[-1].stop == m and ds[-1].is_final
            for a, b in zip(ds, ds[1:]):
                assert a.stop == b.start and a.start % 1024 == 0
            assert all(s.out_start == 3 * s.start // 4 for s in ds)


def _batch_case(count, seed, corrupt):
    """count strings (log-uniform lengths <= 4096), their bytes, texts; `corrupt`: strings that
    get a bad char, plus one truncated (len % 4 != 0) string."""
    L = synth.loguniform_lengths(count, hi=4096, seed=seed)
    off = synth.offsets(L)
    x = synth.data(int(off[-1]), seed=seed)
    enc, eoff = oracle.encode_batch(x, off)
    texts = [enc[eoff[i]: eoff[i + 1]].copy() for i in range(count)]
    for i in corrupt:
        if texts[i].size:
            texts[i][(7 * i) % texts[i].size] = ord("*")
    if count > 9 and texts[9].size:
        texts[9] = texts[9][:-1]
    toff = synth.offsets(np.array([t.size for t in texts], dtype=np.int64))
    return x, off, enc, eoff, np.concatenate(texts) if texts else np.zeros(0, np.uint8), toff


def _batch_worker(rank, world, port, count, seed, corrupt):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        codec = OracleChunkCodec()
        x, off, enc, eoff, text, toff = _batch_case(count, seed, corrupt)
        # encode: shard the input strings by cumulative input bytes; outputs concatenate to the whole
        sh = b64dist.batch_shard(off, world, rank)
        out, oo = b64dist.encode_batch_sharded(torch.from_numpy(x[sh.byte_start: sh.byte_stop].copy()),
                                               torch.from_numpy(off[sh.start: sh.stop + 1] - sh.byte_start), codec)
        parts = [None] * world
        dist.all_gather_object(parts, (sh.start, out.numpy()[: int(oo[-1])].tobytes()))
        assert b"".join(p[1] for p in sorted(parts)) == enc.tobytes()
        # decode: shard the texts by cumulative text bytes
        ds = b64dist.batch_shard(toff, world, rank)
        out, oo, st, err, olen, first = b64dist.decode_batch_sharded(
            torch.from_numpy(text[ds.byte_start: ds.byte_stop].copy()),
            torch.from_numpy(toff[ds.start: ds.stop + 1] - ds.byte_start), ds, codec)
        rout, roo, rst, rerr, rolen = oracle.decode_batch(text, toff)
        assert np.array_equal(st.numpy(), rst[ds.start: ds.stop])
        assert np.array_equal(err.numpy(), rerr[ds.start: ds.stop])
        assert np.array_equal(olen.numpy(), rolen[ds.start: ds.stop])
        o = out.numpy()
        for j, i in enumerate(range(ds.start, ds.stop)):
            assert np.array_equal(o[oo[j]: oo[j] + olen[j]], rout[roo[i]: roo[i] + rolen[i]]), i
        bad = np.nonzero(rst != 0)[0]
        assert first == (int(bad[0]) if bad.size else -1), (rank, first)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,count,corrupt", [(2, 3000, (17, 2500, 2999)), (3, 2000, (1500,)),
                                                 (2, 500, ()), (3, 2, (1,))])
def test_batch_sharded_gloo(world, count, corrupt):
    """configs[3]'s multi-GPU form: strings cut by cumulative bytes, per-string
    results local and equal to the whole batch's, first failing string via one all_reduce(MIN)
    (string 9 is truncated when count > 9: status LENGTH)."""
    mp.spawn(_batch_worker, args=(world, _free_port(), count, count, corrupt), nprocs=world, join=True)


def test_batch_shard_arithmetic():
    """Shards tile the string range in order and balance BYTES: each rank's bytes are within one
    string length of total / world; empty batches, single strings and zero-length strings."""
    rng = np.random.default_rng(3)
    for count in (0, 1, 2, 7, 1000):
        L = np.where(rng.random(count) < 0.2, 0, synth.loguniform_lengths(count, seed=count))
        off = synth.offsets(L.astype(np.int64)) + 5  # any base
        for world in (1, 2, 3, 8):
            sh = [b64dist.batch_shard(off, world, r) for r in range(world)]
            assert sh[0].start == 0 and sh[-1].stop == count
            for a, b in zip(sh, sh[1:]):
                assert a.stop == b.start and a.byte_stop == b.byte_start
            total = int(off[-1] - off[0])
            longest = int(L.max()) if count else 0
            for s_ in sh:
                assert abs((s_.byte_stop - s_.byte_start) - total / world) <= longest + 1
