"""Edge-list ingestion (SPEC S:110-118 load_edge_list): host parsing only."""
import numpy as np
import pytest

import oracle
from paper_1503_04359_b200.edgelist import load_edge_list
from tests import graphs


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_spec_examples(tmp_path):
    uv, n, ids = load_edge_list(_write(tmp_path, "a.txt", "0 1\n1 2\n"))
    assert n == 3 and uv.tolist() == [[0, 1], [1, 2]]
    uv, n, ids = load_edge_list(_write(tmp_path, "b.txt", "# comment\n5 9\n"))
    assert n == 2 and uv.tolist() == [[0, 1]] and ids.tolist() == [5, 9]


def test_g1_round_trip_degree_sequence(tmp_path):
    n0, e = graphs.g1()
    text = "".join(f"{u} {v}\n" for u, v in np.asarray(e).reshape(-1, 2))
    uv, n, _ = load_edge_list(_write(tmp_path, "g1.txt", text))
    g = oracle.build_csr(n, uv)
    assert n == n0 and sorted(g.degree().tolist(), reverse=True) == [3, 2, 2, 1, 1, 1]


def test_errors_and_empty(tmp_path):
    with pytest.raises(ValueError, match=":3:"):
        load_edge_list(_write(tmp_path, "bad.txt", "0 1\n% c\nx y\n"))
    with pytest.raises(ValueError, match=":1:"):
        load_edge_list(_write(tmp_path, "one.txt", "7\n"))
    uv, n, ids = load_edge_list(_write(tmp_path, "empty.txt", ""))
    assert uv.shape == (0, 2) and n == 0
    uv, n, ids = load_edge_list(_write(tmp_path, "pad.txt", "3 4\n"), n_hint=10)
    assert n == 10 and ids[:2].tolist() == [3, 4] and (ids[2:] == -1).all()
    with pytest.raises(ValueError):
        load_edge_list(_write(tmp_path, "pad2.txt", "3 4\n1 2\n"), n_hint=3)


@pytest.mark.parametrize("fmt,dt", [("bin32", np.int32), ("bin64", np.int64)])
def test_binary_equals_text(tmp_path, fmt, dt):
    rng = np.random.default_rng(3)
    e = rng.integers(0, 1 << 20, size=(500, 2))
    p = tmp_path / f"e.{fmt}"
    e.astype(dt).tofile(p)
    ub, nb, ib = load_edge_list(str(p), fmt=fmt)
    ut, nt, it = load_edge_list(_write(tmp_path, "e.txt", "".join(f"{u} {v}\n" for u, v in e)))
    assert nb == nt and np.array_equal(ub, ut) and np.array_equal(ib, it)
    assert np.array_equal(ib[ub], e)          # the mapping restores the file IDs
