"""On-device test problems (kp_generate_test_problems, make_test_problem of
deblur.cpp:201-229 for a batch): the mt19937_64 stream bit for bit against
the host Rng (deblur.cpp:24-42), the normals, blob image, b_true and noise
against the host generator to the last bits, and the C4 pipeline (discrepancy
lambda + batched PCG) unchanged on device-generated images."""
import ctypes as C

import numpy as np
import pytest

import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P

pytestmark = pytest.mark.gpu


def test_mt19937_64_stream_bit_identical():
    seeds = [0, 1, 5000, 2**63 + 12345]
    count = 1000
    raw = P.rng_raw_device(seeds, count)
    for s, row in zip(seeds, raw):
        want = np.empty(count)
        P.lib().kpg_rng_uniforms(C.c_uint64(s), C.c_long(count), 0.0, 1.0, want.ctypes.data)
        got = (row >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        assert np.array_equal(got, want)  # uniforms = the reference's, bit for bit


@pytest.mark.parametrize("n,levels", [(64, [0.01, 0.05]), (96, [0.001, 0.0, 0.02])])
def test_device_problems_match_host_generator(n, levels):
    psf = P.make_psf("gaussian", 17, sigma=2.5)
    a, _ = P.psf_to_kronsum(psf, n)
    seeds = [4000 + i for i in range(len(levels))]
    nseeds = [5000 + i for i in range(len(levels))]
    x, b, e, norms = P.make_test_problems_device(a, seeds, nseeds, levels)
    for i, lv in enumerate(levels):
        tp = P.make_test_problem(P.blob_image(n, seeds[i]), psf, lv, nseeds[i], a=a)
        assert np.allclose(x[i], tp.x_true, rtol=0, atol=1e-15)
        nb = np.linalg.norm(tp.b)
        assert np.linalg.norm(b[i] - tp.b) <= 1e-13 * nb
        if lv == 0.0:
            assert not np.any(e[i]) and norms[i] == 0.0
        else:
            assert np.linalg.norm(e[i] - tp.noise) <= 1e-12 * np.linalg.norm(tp.noise)
            assert norms[i] == pytest.approx(np.linalg.norm(tp.noise), rel=1e-12)
    # the normals themselves: within a few ulp of Rng::normal
    g_host = P.rng_normals(nseeds[0], n * n)
    scale = levels[0] * np.linalg.norm(b[0] - e[0]) / np.linalg.norm(g_host)
    assert np.allclose(e[0] / scale, g_host, rtol=1e-12, atol=1e-15)


def test_c4_pipeline_on_device_generated_images():
    from paper_2311_15393_b200.batch import C4Shard
    sh = C4Shard(n=128)
    ids = list(range(6))
    x, b, e, norms = P.make_test_problems_device(sh.a, [4000 + i for i in ids], [5000 + i for i in ids],
                                                 [[0.001, 0.01, 0.05][i % 3] for i in ids])
    probs = {i: sh.problem(i) for i in ids}
    host = sh.solve_batch(ids, probs)
    dev = sh.solve_arrays(ids, b, x, list(norms), [[0.001, 0.01, 0.05][i % 3] for i in ids])
    for rh, rd in zip(host, dev):
        assert rd.lam == pytest.approx(rh.lam, rel=1e-9)
        assert abs(rd.iterations - rh.iterations) <= 2
        assert abs(rd.rel_err - rh.rel_err) <= 1e-6
