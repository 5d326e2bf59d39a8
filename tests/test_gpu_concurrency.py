"""Stream-ordered launches on independent state blocks (include/fsmc.h: the
launch bookkeeping lives in each fsmc_state's own work[] words).  Two batches
advanced concurrently on two streams through the C ABI must equal the same
batches run one after the other."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fm():
    import paper_2503_17405_b200 as fm
    return fm


def _launch(fm, bundle, target, batch, n, out, stream, window=0, parts=1, draws=None):
    from paper_2503_17405_b200 import _lib
    K = bundle.fsm.n_states
    order = (ctypes.c_int32 * K)(*([K] + list(range(1, K))))
    lib = _lib.lib()
    args = (ctypes.byref(batch.kernel), ctypes.byref(target.struct()), ctypes.byref(batch.struct()),
            n, _lib.BUNDLED, order, 1 << 62, 0, ctypes.byref(out))
    if window:
        _lib.check(lib.fsmc_run_windowed_overlap(*args, window, draws.data_ptr(), 0, parts,
                                                 stream.cuda_stream), "windowed")
    else:
        _lib.check(lib.fsmc_run(*args, 0, stream.cuda_stream), "run")


def _outputs(batch, n, d):
    import torch
    from paper_2503_17405_b200 import _lib
    s = torch.zeros((n, batch.m, d), dtype=torch.float64, device="cuda")
    c = torch.zeros((1, n, batch.m), dtype=torch.int32, device="cuda")
    o = _lib.Outputs()
    o.samples, o.loop_counts, o.sample_ticks = s.data_ptr(), c.data_ptr(), None
    return s, c, o


def test_two_batches_on_two_streams_equal_serial_runs(fm):
    import torch
    bundle = fm.drmh_kernel(100, 0.1)
    target = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
    m_a, m_b, n, d, W = 6000, 5000, 60, 10, 660
    res = {}
    for mode in ("serial", "concurrent"):
        a = fm.init_batch(bundle, target, m_a, 21)
        b = fm.init_batch(bundle, target, m_b, 22)
        sa, ca, oa = _outputs(a, n, d)
        sb, cb, ob = _outputs(b, n, d)
        draws = torch.empty(m_b * W + 32, dtype=torch.float64, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        torch.cuda.synchronize()
        _launch(fm, bundle, target, a, n, oa, s1)
        if mode == "serial":
            s1.synchronize()
        _launch(fm, bundle, target, b, n, ob, s2, window=W, parts=4, draws=draws)
        torch.cuda.synchronize()
        res[mode] = [t.cpu().numpy() for t in (sa, ca, sb, cb)]
        assert (res[mode][1] > 0).all() and (res[mode][3] > 0).all()
    for x, y in zip(res["serial"], res["concurrent"]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("m", [4096, 16384])
def test_streamed_host_output_equals_device_output(fm, m):
    """output="numpy" streams finished chain parts to pinned host memory
    during the run (fsmc_run_egress); the samples and ledger equal the
    device-resident run's."""
    bundle, target = fm.nuts_kernel(0.05, 10), fm.equicorrelated_gaussian_target(100, 0.99)
    n = 12
    a, la = fm.run_fsm_batched(bundle, target, fm.init_batch(bundle, target, m, 4), n,
                               step_variant="bundled", output="numpy", surplus=False)
    b, lb = fm.run_fsm_batched(bundle, target, fm.init_batch(bundle, target, m, 4), n,
                               step_variant="bundled", output="torch", surplus=False)
    assert np.array_equal(a, b.cpu().numpy())
    assert np.array_equal(la.iter_counts, lb.iter_counts.cpu().numpy())


def test_streamed_host_output_of_the_prior_transform_rounds(fm):
    """The batched prior-transform rounds (C4's path) send each round's
    finished sample rows of every chain part to pinned host memory while the
    rounds continue; the result equals the device-resident run's."""
    bundle, target = fm.elliptical_kernel(), fm.gp_classification_target(256)
    m, n = 600, 15
    runs = []
    for output in ("numpy", "torch"):
        s, led = fm.run_fsm_batched(bundle, target, fm.init_batch(bundle, target, m, 8), n,
                                    step_variant="amortized", output=output, surplus=False,
                                    prior_transform="dmma", prior_parts=3)
        runs.append((np.asarray(s) if output == "numpy" else s.cpu().numpy(),
                     np.asarray(led.iter_counts) if output == "numpy" else led.iter_counts.cpu().numpy()))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("parts", [1, 3, 12, 0])
def test_streamed_host_output_of_windowed_runs(fm, parts):
    """The windowed DRMH run (C2's path) copies each chain part's finished
    sample and count rows to pinned host memory at its progress checks
    (per-part pitched copies; one range in the pipelined mode); the host
    result equals the device-resident run's."""
    bundle, target = fm.drmh_kernel(100, 0.1), fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
    m, n = 6000, 40
    runs = []
    for output in ("numpy", "torch"):
        s, led = fm.run_fsm_batched(bundle, target, fm.init_batch(bundle, target, m, 21), n,
                                    step_variant="bundled", output=output, surplus=False,
                                    draw_window=1100, draw_parts=parts)
        to_np = (lambda v: np.asarray(v)) if output == "numpy" else (lambda v: v.cpu().numpy())
        runs.append((to_np(s), to_np(led.iter_counts), to_np(led.loop_exec_counts[2])))
    for x, y in zip(*runs):
        assert np.array_equal(x, y)
