"""GPU parity for the stream-K schedule of the tcgen05 pair kernel.

Stream-K deals the (tile, k-block) units of a GEMM out evenly over the
clusters; a tile cut between clusters is finished by the cluster holding its
last k-blocks, which adds the other clusters' FP32 partial tiles (fixed order)
before the epilogue (bias, FP32 C, fused Q node, counters). Only the FP32
summation order changes, so on an exact operand grid (every partial sum exact
in FP32) the results equal the exact result bit for bit; on N(0,1) data they
stay within the stated tolerance tau = 1e-6 * (|A||B|)_ij.
"""
import os
import threading

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
TAU = 1e-6
KNOBS = ("FP8B_GEMM_SK", "FP8B_GEMM_NB", "FP8B_GEMM_SPLITK")


@pytest.fixture(scope="module")
def fp8():
    import paper_1905_12334_b200 as F
    F.init()
    return F


@pytest.fixture
def env():
    old = {k: os.environ.get(k) for k in KNOBS}
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _codes_dev(c):
    import torch
    return torch.from_numpy(np.ascontiguousarray(c).astype(np.uint8)).to("cuda")


def _grid_operands(rng, m, k, n):
    A = O.quantize((rng.integers(-2, 3, m * k) * 0.5).astype(np.float32))[0].reshape(m, k)
    B = O.quantize((rng.integers(-2, 3, k * n) * 0.25).astype(np.float32))[0].reshape(k, n)
    return A, B


# (m, k, n): ragged in every dimension; k-block counts from 3 to 97 so that
# tiles are cut into 1..many pieces, some clusters hold only a middle piece
SHAPES = [(1000, 1536, 1100), (512, 12416, 768), (2048, 384, 2560), (300, 4096, 520),
          (4096, 2048, 4096), (5120, 1024, 4352)]


@pytest.mark.parametrize("sk", ["1", "2"])  # 1: whole waves data-parallel + stream-K rest; 2: all stream-K
@pytest.mark.parametrize("nb", ["1", "2"])
@pytest.mark.parametrize("m,k,n", SHAPES, ids=lambda v: str(v))
@pytest.mark.parametrize("out", ["f32+fp8", "codes", "f32+fp16sr"])
def test_streamk_exact_grid(fp8, env, sk, nb, m, k, n, out):
    import torch
    env["FP8B_GEMM_SK"] = sk
    env["FP8B_GEMM_NB"] = nb
    env["FP8B_GEMM_SPLITK"] = "1"
    rng = np.random.default_rng(m + k + n)
    A, B = _grid_operands(rng, m, k, n)
    bias = (rng.integers(-8, 8, n) * 0.125).astype(np.float32)
    bias[3::61] = 60000.0  # overflow columns
    out_fmt, out_mode = ("fp16", "stochastic") if out == "f32+fp16sr" else ("fp8", "nearest-even")
    cnt = fp8.Counters()
    c, cq = fp8.gemm_codes(_codes_dev(A), _codes_dev(B), m, n, k, "fp8", engine="tensor",
                           want_c=out != "codes", bias=torch.from_numpy(bias).cuda(),
                           out_fmt=out_fmt, out_mode=out_mode, out_seed=5, out_counters=cnt)
    da = O.dequantize(A).astype(np.float64).reshape(m, k)
    db = O.dequantize(B).astype(np.float64).reshape(k, n)
    y = ((da @ db).astype(np.float32) + bias[None, :]).astype(np.float32)
    if c is not None:
        np.testing.assert_array_equal(c.cpu().numpy(), y)
    codes, k_ = O.quantize(y, out_fmt, out_mode, 5, bits="counter")
    got = cq.cpu().numpy()
    got = got.view(np.uint16) if out_fmt == "fp16" else got
    np.testing.assert_array_equal(got, codes.astype(got.dtype))
    assert cnt.values() == tuple(int(v) for v in k_)


@pytest.mark.parametrize("a_major", ["k", "m"])
@pytest.mark.parametrize("nb", ["1", "2"])
@pytest.mark.parametrize("sk", ["1", "2"])
def test_streamk_tolerance_and_determinism(fp8, env, a_major, nb, sk):
    """N(0,1) E5M2 operands, long K: within tau of the exact sum; two runs are
    bitwise identical (the partial-tile sum order is fixed by the unit split,
    not by which cluster arrives first)."""
    import torch
    env["FP8B_GEMM_SK"] = sk
    env["FP8B_GEMM_NB"] = nb
    m, k, n = 1536, 8192, 1024
    x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
    fp8.fill_synthetic(x, "normal", 17, 1.0)
    qa, qb = fp8.quantize(x[: m * k]), fp8.quantize(x[m * k:])
    c1, _ = fp8.gemm_codes(qa.codes, qb.codes, m, n, k, "fp8", a_major=a_major, engine="tensor")
    c2, _ = fp8.gemm_codes(qa.codes, qb.codes, m, n, k, "fp8", a_major=a_major, engine="tensor")
    assert torch.equal(c1.view(torch.int32), c2.view(torch.int32))
    da = fp8.dequantize(qa).double()
    da = da.reshape(m, k) if a_major == "k" else da.reshape(k, m).t()
    db = fp8.dequantize(qb).double().reshape(k, n)
    err = (c1.double() - da @ db).abs()
    assert bool((err <= TAU * (da.abs() @ db.abs()) + 1e-30).all())


def test_streamk_concurrent_streams(fp8, env):
    """Two stream-K GEMMs in flight at once on two streams (as the dense step's
    parallel graph branches run them): neither relies on all its clusters being
    resident, so both finish and both are exact."""
    import torch
    env["FP8B_GEMM_SK"] = "2"
    rng = np.random.default_rng(3)
    jobs = []
    for (m, k, n) in [(2048, 4096, 2560), (1024, 8192, 3072)]:
        A, B = _grid_operands(rng, m, k, n)
        da = O.dequantize(A).astype(np.float64).reshape(m, k)
        db = O.dequantize(B).astype(np.float64).reshape(k, n)
        jobs.append((m, k, n, _codes_dev(A), _codes_dev(B), (da @ db).astype(np.float32)))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [None, None]
    torch.cuda.synchronize()
    for rep in range(5):
        for i, (m, k, n, a, b, _) in enumerate(jobs):
            with torch.cuda.stream(streams[i]):
                outs[i], _ = fp8.gemm_codes(a, b, m, n, k, "fp8", engine="tensor",
                                            stream=streams[i])
        done = threading.Event()
        t = threading.Thread(target=lambda: (torch.cuda.synchronize(), done.set()), daemon=True)
        t.start()
        assert done.wait(60), "stream-K GEMMs on two streams did not finish"
        for i, (_, _, _, _, _, y) in enumerate(jobs):
            np.testing.assert_array_equal(outs[i].cpu().numpy(), y)


def test_streamk_in_cuda_graph(fp8, env):
    """Captured once, replayed many times: the workspace flags and the cluster
    ticket reset themselves, so every replay is exact."""
    import torch
    env["FP8B_GEMM_SK"] = "2"
    rng = np.random.default_rng(9)
    m, k, n = 1000, 3072, 1300
    A, B = _grid_operands(rng, m, k, n)
    a, b = _codes_dev(A), _codes_dev(B)
    da = O.dequantize(A).astype(np.float64).reshape(m, k)
    db = O.dequantize(B).astype(np.float64).reshape(k, n)
    y = (da @ db).astype(np.float32)
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fp8.gemm_codes(a, b, m, n, k, "fp8", engine="tensor", c=c, stream=s)  # warm up
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fp8.gemm_codes(a, b, m, n, k, "fp8", engine="tensor", c=c, stream=s)
    for _ in range(20):
        c.zero_()
        g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(c.cpu().numpy(), y)
