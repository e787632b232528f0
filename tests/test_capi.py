"""C-ABI boundary checks that run without a GPU: the library loads, exports
every function include/ihs_gpu.h declares, and its host-side logic (tuning
scalars, seeds, sparse Fisher-Yates, synthetic data) matches the oracle."""
import ctypes
import pathlib
import re

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "ihs_gpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(ihs_\w+)\s*\(", text))
    names.discard("ihs_sketch_override_fn")
    return sorted(n for n in names if not n.endswith("_fn"))


def test_library_exports_every_declared_symbol(ihs):
    from paper_2006_05874_b200 import _lib

    L = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    # the Python mirror binds exactly the declared entry points
    assert set(declared_functions()) == set(_lib.EXPORTED_SYMBOLS)


def test_version_and_launch_counter(ihs):
    from paper_2006_05874_b200._lib import lib

    assert b"sm_100a" in lib().ihs_gpu_version()
    assert ihs.kernel_launch_count() >= 0


def test_tuning_matches_oracle(ihs, O):
    for lam, Lam in [(0.5, 2.0), (1.0, 1.0), (0.2, 1.7), (1e-3, 3.9)]:
        a = ihs.rates_from_bounds(lam, Lam)
        b = O.rates_from_bounds(lam, Lam)
        assert a.__dict__ == b.as_dict()
    for rho in (0.01, 0.1, 0.18):
        assert ihs.gaussian_targets(rho, 0.01) == O.gaussian_targets(rho, 0.01)
        assert ihs.srht_targets(rho) == O.srht_targets(rho)
    with pytest.raises(ihs.OutOfValidityRange):
        ihs.gaussian_targets(0.19, 0.01)
    with pytest.raises(ihs.InvalidInput):
        ihs.gaussian_targets(-0.1, 0.01)
    with pytest.raises(ihs.InvalidInput):
        ihs.srht_targets(1.0)
    with pytest.raises(ihs.InvalidInput):
        ihs.rates_from_bounds(2.0, 1.0)
    ihs.gaussian_targets(0.19, 0.01, False)


def test_seeds_and_pow2(ihs, O):
    for s, t in [(0, 0), (5, 1), (2**64 - 1, 3), (123456789, 1000)]:
        assert ihs.derive_seed(s, t) == O.derive_seed(s, t)
    for n in (1, 2, 3, 1000, 1024, 10**6):
        assert ihs.next_pow2(n) == O.next_pow2(n)


@pytest.mark.parametrize("n,m", [(16, 16), (128, 100), (1024, 1), (1 << 20, 3000), (1 << 22, 65536), (1000003, 77)])
def test_sparse_fisher_yates_is_the_reference_sample(ihs, O, n, m):
    s = O.derive_seed(O.derive_seed(42, m), 2)
    assert np.array_equal(ihs.sample_without_replacement(s, n, m), O.sample_without_replacement(s, n, m))


@pytest.mark.parametrize("n,d,frac", [(5000, 40, 0.01), (70000, 6, 0.0), (1000, 1000, 0.0)])
def test_synth_generator_matches_oracle(ihs, O, n, d, frac):
    A, b, xt = ihs.synth_generate(n, d, decay=0.97, noise_std=0.1, outlier_frac=frac, data_seed=11)
    A2, b2, xt2 = O.synth(n, d, decay=0.97, noise_std=0.1, outlier_frac=frac, data_seed=11)
    assert np.array_equal(A, A2) and np.array_equal(b, b2) and np.array_equal(xt, xt2)


def test_synth_row_ranges_compose(ihs):
    n, d = 140000, 3
    A, b, _ = ihs.synth_generate(n, d, decay=0.9, data_seed=2)
    A1, b1, _ = ihs.synth_generate(n, d, decay=0.9, data_seed=2, row0=50000, rows=70000)
    assert np.array_equal(A[50000:120000], A1) and np.array_equal(b[50000:120000], b1)


def test_newton_decrement_host(ihs):
    assert ihs.newton_decrement([1.0, 2.0], [3.0, 4.0]) == 0.5 * 11.0
    with pytest.raises(ihs.NumericalBreakdown):
        ihs.newton_decrement(np.ones(3), -np.ones(3))
    assert ihs.newton_decrement([1e-20], [-1e-20]) == 0.0
