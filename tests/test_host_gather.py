"""_hps_host.gather_rows (host-side gather of a {leaf id: (m,)} load mapping, the reference's
g convention, solver.py:241-253): same table as the numpy path, -1 / position protocol for
values the fast path does not take, KeyError for a missing leaf."""
import numpy as np
import pytest

from paper_1612_02736_b200 import _ext


@pytest.fixture(scope="module")
def host():
    mod = _ext.host_module()
    if mod is None:
        pytest.skip("no host compiler: the numpy gather path is used")
    return mod


@pytest.mark.parametrize("threads", [1, 3])
def test_gather_matches_concatenate(host, threads):
    rng = np.random.default_rng(0)
    n, m = 1500, 196  # > 1 MiB: the threaded copy path
    tab = rng.standard_normal((n, m))
    ids = [int(i) for i in rng.permutation(n) + 11]
    g = {nid: tab[r] for r, nid in enumerate(ids)}
    out = np.empty((n, m))
    assert host.gather_rows(g, ids, out, threads) == -1
    assert np.array_equal(out, tab)


def test_generic_mapping_and_bad_values(host):
    from collections import UserDict
    m = 5
    ids = [3, 1, 2]
    g = UserDict({1: np.arange(5.0), 2: np.ones(5), 3: np.full(5, 7.0)})
    out = np.empty((3, m))
    assert host.gather_rows(g, ids, out, 1) == -1
    assert np.array_equal(out, np.stack([g[3], g[1], g[2]]))
    # values the fast path leaves to the caller: wrong length, lists, float32, strided views
    for bad in (np.ones(4), [1.0] * 5, np.ones(5, dtype=np.float32), np.ones(10)[::2]):
        g2 = dict(g)
        g2[1] = bad
        assert host.gather_rows(g2, ids, out, 1) == 1
    with pytest.raises(KeyError):
        host.gather_rows({1: np.ones(5)}, ids, out, 1)
    with pytest.raises(ValueError):
        host.gather_rows(dict(g), ids, np.empty((2, m)), 1)
