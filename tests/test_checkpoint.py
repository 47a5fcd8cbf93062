"""CKPTIMG1 checkpoint layer against images written by
the real reference (tests/golden/make_ckpt_golden.py).

CPU tests: image format, checksum/structure errors, atomic commits, raw
payloads, and the lossy fixtures re-decoded by the oracle.  GPU tests: lossy
images byte-identical to the reference's, device decode, the asynchronous
checkpointer overlapping with device work, recover().  Mirrors the
reference's test_checkpoint.py coverage (image round trip, corruption,
commit atomicity, raw/lossy recovery)."""

import os
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1805_07384_b200 import checkpoint as ck
from paper_1805_07384_b200.errors import CheckpointFailedError, ParameterError, UnrecoverableImageError
from tests.conftest import ROOT

CKG = os.path.join(ROOT, "tests", "golden", "ckpt_golden.npz")


@pytest.fixture(scope="module")
def ckg():
    return np.load(CKG, allow_pickle=False)


def _names(z, kind):
    return sorted({k.split("/")[0] for k in z.files if k.startswith(kind)})


def _cfg(lc, mode, param):
    return {0: lc.CompressorConfig.absolute, 1: lc.CompressorConfig.value_range_relative,
            2: lc.CompressorConfig.fixed_psnr}[int(mode)](float(param))


def test_raw_images_byte_identical(ckg):
    for name in _names(ckg, "raw"):
        x = ckg[name + "/x"]
        it = int(ckg[name + "/meta"][0])
        img, cost = ck.checkpoint_traditional(SimpleNamespace(x=x, iteration=it), ck.StorageTarget(), commit=False)
        assert img.to_bytes() == ckg[name + "/image"].tobytes(), name
        assert cost.payload_bytes == img.nbytes and cost.t_compress == 0.0
        back = ck.decode_payload(ck.CheckpointImage.from_bytes(ckg[name + "/image"].tobytes()))
        assert back.dtype == np.float64 and np.array_equal(back.view(np.int64), x.view(np.int64))


def test_image_parse_and_corruption(ckg):
    blob = ckg["lossy_rel4/image"].tobytes()
    img = ck.CheckpointImage.from_bytes(blob)
    assert img.iteration == 42 and img.kind == ck.PAYLOAD_LOSSY and img.to_bytes() == blob
    head = len(ck.IMAGE_MAGIC) + 29
    bad = [b"XKPTIMG1" + blob[8:],                              # magic
           blob[:8] + (2).to_bytes(4, "little") + blob[12:],     # version
           blob[:-1],                                            # length
           blob[:head] + bytes([blob[head] ^ 1]) + blob[head + 1:],  # checksum
           blob[:8]]                                             # truncated header
    for b in bad:
        with pytest.raises(UnrecoverableImageError):
            ck.CheckpointImage.from_bytes(b)
    tampered = ck.CheckpointImage(iteration=1, kind=ck.PAYLOAD_RAW, payload=b"\0" * 8, checksum=0)
    with pytest.raises(UnrecoverableImageError):
        ck.decode_payload(tampered)
    with pytest.raises(ParameterError):
        ck.CheckpointImage(iteration=0, kind=7, payload=b"", checksum=0)


def test_storage_target_atomic_commit(tmp_path, ckg):
    path = tmp_path / "ckpt.img"
    t = ck.StorageTarget(write_bandwidth=1e9, read_bandwidth=2e9, path=path)
    assert t.load_last() is None
    a = ck.CheckpointImage.from_bytes(ckg["raw_small/image"].tobytes())
    t.commit(a)
    assert path.read_bytes() == a.to_bytes() and not (tmp_path / "ckpt.img.tmp").exists()
    assert t.load_last().to_bytes() == a.to_bytes()
    assert t.write_time(1e9) == 1.0 and t.read_time(2e9) == 1.0
    broken = ck.StorageTarget(path=tmp_path / "missing_dir" / "ckpt.img")
    with pytest.raises(CheckpointFailedError):
        broken.commit(a)
    assert broken.load_last() is None
    mem = ck.StorageTarget()
    mem.commit(a)
    assert mem.load_last() is a
    with pytest.raises(ParameterError):
        ck.StorageTarget(write_bandwidth=0)


def test_lossy_fixtures_pinned_by_oracle(ckg):
    """The reference's lossy images decode to the reference recon through the CPU oracle."""
    from oracle import oracle as orc
    for name in _names(ckg, "lossy"):
        img = ck.CheckpointImage.from_bytes(ckg[name + "/image"].tobytes())
        blk = orc.from_bytes(img.payload)
        rec = orc.decompress(blk)
        assert np.array_equal(rec.view(np.int64), ckg[name + "/recon"].view(np.int64)), name


def test_recover_raw_with_and_without_rebuild(ckg):
    img = ck.CheckpointImage.from_bytes(ckg["raw_small/image"].tobytes())
    state, cost = ck.recover(img, "cg", None, None, None, None, target=ck.StorageTarget(read_bandwidth=1e6))
    assert state.iteration == 7 and np.array_equal(state.x, ckg["raw_small/x"])
    assert cost.t_decompress == 0.0 and cost.t_read == img.nbytes / 1e6
    seen = {}

    def rebuild(method, a, m, b, x, iteration, config):
        seen.update(method=method, iteration=iteration, n=len(x))
        return "rebuilt"

    state, _ = ck.recover(img, "jacobi", 1, 2, 3, "cfg", rebuild=rebuild)
    assert state == "rebuilt" and seen == dict(method="jacobi", iteration=7, n=257)


torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def lc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1805_07384_b200 as lc
    return lc


@pytest.mark.gpu
def test_lossy_images_byte_identical(lc, ckg):
    for name in _names(ckg, "lossy"):
        x = ckg[name + "/x"]
        it, _, mode, param = ckg[name + "/meta"]
        want = ckg[name + "/image"].tobytes()
        for xin in (x, torch.from_numpy(x).cuda()):
            img, cost = ck.checkpoint_lossy(SimpleNamespace(x=xin, iteration=int(it)), _cfg(lc, mode, param),
                                            ck.StorageTarget(), commit=False, block_version=1)
            assert img.to_bytes() == want, name
            # the repo's default image (v3 block) decodes to the same reconstruction
            img3, _ = ck.checkpoint_lossy(SimpleNamespace(x=xin, iteration=int(it)), _cfg(lc, mode, param),
                                          ck.StorageTarget(), commit=False)
            assert lc.CompressedBlock.from_bytes(img3.payload).version == 3
            assert np.array_equal(ck.decode_payload(img3).view(np.int64), ckg[name + "/recon"].view(np.int64))
            assert cost.t_compress > 0.0 and cost.payload_bytes == len(want)


@pytest.mark.gpu
def test_decode_payload_device(lc, ckg):
    for name in _names(ckg, "lossy"):
        img = ck.CheckpointImage.from_bytes(ckg[name + "/image"].tobytes())
        ref = ckg[name + "/recon"]
        host = ck.decode_payload(img)
        dev = ck.decode_payload(img, device="cuda")
        assert isinstance(host, np.ndarray) and dev.is_cuda
        assert np.array_equal(host.view(np.int64), ref.view(np.int64)), name
        assert np.array_equal(dev.cpu().numpy().view(np.int64), ref.view(np.int64)), name
        state, cost = ck.recover(img, "cg", None, None, None, None, device="cuda")
        assert state.iteration == img.iteration and cost.t_decompress > 0.0


@pytest.mark.gpu
def test_async_checkpointer_overlaps_and_matches(lc, ckg, tmp_path):
    x0 = torch.from_numpy(ckg["lossy_rel4/x"]).cuda()
    cfg = lc.CompressorConfig.value_range_relative(1e-4)
    target = ck.StorageTarget(path=tmp_path / "async.img")
    x = x0.clone()
    futures, expect = [], []
    with ck.AsyncCheckpointer(cfg, target, max_in_flight=2) as acp:
        for it in range(4):
            expect.append(x.clone())
            futures.append(acp.submit(SimpleNamespace(x=x, iteration=it)))
            x.mul_(1.0001).add_(1e-3)             # the "solver" keeps modifying x meanwhile
        images = [f.result()[0] for f in futures]
    for it, (img, xs) in enumerate(zip(images, expect)):
        sync, _ = ck.checkpoint_lossy(SimpleNamespace(x=xs, iteration=it), cfg, ck.StorageTarget(), commit=False)
        assert img.to_bytes() == sync.to_bytes()
    assert ck.CheckpointImage.from_bytes((tmp_path / "async.img").read_bytes()).iteration == 3
    ref0 = ck.CheckpointImage.from_bytes(ckg["lossy_rel4/image"].tobytes()).payload
    assert lc.CompressedBlock.from_bytes(images[0].payload).payload == lc.CompressedBlock.from_bytes(ref0).payload
