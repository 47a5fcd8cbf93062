"""Multi-rank sharded checkpoint path on CPU with the gloo
backend, world_size 2: slab bounds, the metadata all-gather + exclusive scan
that places every rank's LCKP0001 blob, concurrent positional writes into one
LCKPSHD1 image, per-rank reads, and the max-over-ranks timing reduction the
bench uses.  Shard blocks come from the CPU oracle (test infrastructure);
the GPU path runs the same functions over NCCL (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1805_07384_b200 import shard  # noqa: E402
from paper_1805_07384_b200.compressor import CompressedBlock  # noqa: E402
from paper_1805_07384_b200.errors import IntegrityError, ParameterError  # noqa: E402

WORLD = 2
N_GLOBAL = 50_001


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global_vector():
    r = np.random.default_rng(11)
    x = np.cumsum(r.normal(0, 1, N_GLOBAL))
    x[::7919] += 1e4
    return x


def _oracle_block(x, eb_rel):
    from oracle import oracle as orc
    d = orc.compress(x, "value_range_relative", eb_rel)
    return CompressedBlock(n=d["n"], eb_abs=d["eb_abs"], value_range=d["value_range"],
                           first_value=d["first_value"], code_lengths=d["code_lengths"],
                           payload=d["payload"], payload_bits=d["payload_bits"],
                           escape_indices=d["escape_indices"], escape_values=d["escape_values"])


def _worker(rank, port, path, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        x = _global_vector()
        lo, hi = shard.shard_bounds(N_GLOBAL, WORLD, rank)
        blk = _oracle_block(x[lo:hi], 1e-5)
        blob = blk.to_bytes()
        layout = shard.gather_layout(shard.block_meta(blk, blob))
        if os.path.exists(path) and rank == 0:
            assert open(path, "rb").read() == b"previous image"
        shard.commit_sharded(path, rank, blob, layout)     # atomic: tmp + fsync + replace
        assert not os.path.exists(path + ".tmp")
        slowest = shard.max_over_ranks(10.0 + rank)
        # every rank can read every shard; its own is byte-identical
        got = [shard.read_shard(path, r) for r in range(WORLD)]
        assert got[rank].to_bytes() == blob
        np.save(os.path.join(outdir, f"r{rank}.npy"),
                np.array([layout.offsets[rank], layout.nbytes[rank], layout.total_bytes, slowest, lo, hi]))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_partition():
    for n in (0, 1, 7, 1000, 2 ** 20 + 3):
        for world in (1, 2, 3, 8):
            parts = [shard.shard_bounds(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ParameterError):
        shard.shard_bounds(10, 2, 2)


def test_layout_exclusive_scan():
    meta = np.array([[10, 80, 0, 100, 1], [12, 90, 1, 120, 2], [9, 70, 0, 90, -3]])
    lay = shard.layout_from_meta(meta)
    h = shard.header_bytes(3)
    assert lay.offsets == (h, h + 100, h + 220) and lay.total_bytes == h + 310
    assert shard.decode_header(shard.encode_header(lay)).offsets == lay.offsets
    assert shard.decode_header(shard.encode_header(lay)).checksums == (1, 2, 2 ** 64 - 3)
    with pytest.raises(IntegrityError):
        shard.decode_header(b"LCKPSHD0" + shard.encode_header(lay)[8:])


def test_gloo_world2_sharded_image(tmp_path):
    path = str(tmp_path / "sharded.img")
    with open(path, "wb") as f:                          # the image a commit replaces
        f.write(b"previous image")
    mp.spawn(_worker, args=(_free_port(), path, str(tmp_path)), nprocs=WORLD, join=True)
    rows = [np.load(str(tmp_path / f"r{r}.npy")) for r in range(WORLD)]
    assert [int(r[3]) for r in rows] == [11, 11]                       # max over ranks
    assert int(rows[0][0]) == shard.header_bytes(WORLD)
    assert int(rows[1][0]) == int(rows[0][0] + rows[0][1])              # exclusive scan
    assert os.path.getsize(path) == int(rows[0][2])
    # the sharded image holds exactly the per-slab blocks of the global vector
    x = _global_vector()
    from oracle import oracle as orc
    for r in range(WORLD):
        lo, hi = int(rows[r][4]), int(rows[r][5])
        blk = shard.read_shard(path, r)
        assert blk.to_bytes() == _oracle_block(x[lo:hi], 1e-5).to_bytes()
        d = orc.from_bytes(blk.to_bytes())
        rec = orc.decompress(d)
        assert np.all(np.abs(rec - x[lo:hi]) <= blk.eb_abs)


def test_corrupt_shard_detected(tmp_path):
    """A flipped payload byte (a torn write over stale bytes) fails the per-shard
    BLAKE2b-64 check instead of decoding to a wrong vector."""
    x = _global_vector()[:5000]
    blk = _oracle_block(x, 1e-4)
    blob = blk.to_bytes()
    layout = shard.layout_from_meta(shard.block_meta(blk, blob)[None, :])
    path = str(tmp_path / "one.img")
    shard.prepare_image(path, layout)
    shard.write_shard(path, 0, blob, layout)
    assert shard.read_shard(path, 0).to_bytes() == blob
    raw = bytearray(open(path, "rb").read())
    raw[-10] ^= 0x40
    open(path, "wb").write(bytes(raw))
    with pytest.raises(IntegrityError, match="checksum"):
        shard.read_shard(path, 0)
