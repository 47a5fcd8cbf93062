"""Distortion statistics on the device:
measured_psnr and error_identity_check through lc_error_stats_f64 against the
reference's numpy formulas (compressor.py:81-94, 443-460).  Value range and
max error are exact; MSE is a compensated sum, within 1e-12 relative of
numpy's pairwise sum (written here as the tolerance)."""

import math

import numpy as np
import pytest

from paper_1805_07384_b200.errors import ParameterError, UndefinedPsnrError

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
MSE_RTOL = 1e-12


@pytest.fixture(scope="module")
def lc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1805_07384_b200 as lc
    return lc


def test_measured_psnr_device_matches_numpy(lc):
    rng = np.random.default_rng(7)
    for n in (1, 2, 1000, 1 << 20, (1 << 22) + 3):
        x = np.cumsum(rng.normal(size=n))
        y = x + rng.uniform(-1e-3, 1e-3, n)
        if n == 1:
            x = np.array([0.0, 1.0])[:1]
        ref = None
        try:
            ref = lc.measured_psnr(x, y)
        except UndefinedPsnrError:
            with pytest.raises(UndefinedPsnrError):
                lc.measured_psnr(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
            continue
        for got in (lc.measured_psnr(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()),
                    lc.measured_psnr(x, y, device="cuda")):
            assert math.isclose(got.mse, ref.mse, rel_tol=MSE_RTOL)
            assert math.isclose(got.nrmse, ref.nrmse, rel_tol=MSE_RTOL)
            assert math.isclose(got.psnr_db, ref.psnr_db, rel_tol=MSE_RTOL)


def test_measured_psnr_device_edge_cases(lc):
    x = torch.linspace(0, 1, 1000, dtype=torch.float64, device="cuda")
    same = lc.measured_psnr(x, x.clone())
    assert same.mse == 0.0 and same.psnr_db == math.inf
    with pytest.raises(UndefinedPsnrError):
        lc.measured_psnr(torch.ones(10, dtype=torch.float64, device="cuda"), x[:10])
    with pytest.raises(ParameterError):
        lc.measured_psnr(x, x[:-1])


def test_error_identity_device_matches_host(lc):
    rng = np.random.default_rng(3)
    x = np.cumsum(rng.normal(0, 1, 1 << 18))
    x[::4099] += 1e5                                      # escapes
    for eb in (1e-2, 1e-5):
        blk = lc.compress(x, lc.CompressorConfig.value_range_relative(eb, record_traces=True))
        host = lc.error_identity_check(x, blk)
        dev = lc.error_identity_check(torch.from_numpy(x).cuda(), blk)
        dev2 = lc.error_identity_check(x, blk, device="cuda")
        assert dev == host and dev2 == host
