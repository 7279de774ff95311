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
