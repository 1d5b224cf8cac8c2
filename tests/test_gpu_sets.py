"""Device index sets: enumeration and neighbour tables bit-exact with the reference."""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import hprop_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hp():
    import paper_1403_3511_b200 as hp

    return hp


def test_sizes_match_reference(hp, golden):
    g = golden["sets"]
    for key, val in zip(g["hyp_sizes_keys"], g["hyp_sizes_vals"]):
        dim, bound = map(int, str(key).split("_"))
        assert hp.build_hyperbolic(dim, bound).size == val, key


def test_indices_and_tables_bitexact(hp, golden):
    g = golden["sets"]
    for key in [k for k in g if k.endswith("_indices")]:
        _, kind, dim, bound, _ = key.split("_")
        dim, bound = int(dim), int(bound)
        s = hp.build_hyperbolic(dim, bound) if kind == "hyp" else hp.build_full(dim, bound)
        assert np.array_equal(s.indices, g[key]), key
        base = key[: -len("_indices")]
        for a in range(1, dim + 1):
            d, u = s.neighbor_ordinals(a)
            assert d.dtype == np.int64 and not d.flags.writeable
            assert np.array_equal(d, g[f"{base}_down{a}"]), (key, a)
            assert np.array_equal(u, g[f"{base}_up{a}"]), (key, a)


@pytest.mark.parametrize("dim,bound", [(1, 0), (1, 9), (2, 0), (3, 1), (5, 40), (7, 30), (8, 255), (6, 1023)])
def test_hyperbolic_matches_oracle(hp, dim, bound):
    s = hp.build_hyperbolic(dim, bound)
    ref = O.hyperbolic_indices(dim, bound)
    assert np.array_equal(s.indices, ref)
    tabs = O.neighbor_tables(ref)
    for a in range(1, dim + 1):
        d, u = s.neighbor_ordinals(a)
        assert np.array_equal(d, tabs[a - 1][0]) and np.array_equal(u, tabs[a - 1][1])


def test_custom_set_tables(hp):
    rows = O.hyperbolic_indices(3, 20).tolist()
    s = hp.from_indices(rows)
    assert s.kind == "custom"
    tabs = O.neighbor_tables(np.asarray(sorted(map(tuple, rows)), dtype=np.int64))
    for a in (1, 2, 3):
        d, u = s.neighbor_ordinals(a)
        assert np.array_equal(d, tabs[a - 1][0]) and np.array_equal(u, tabs[a - 1][1])


def test_position_contains_neighbor_api(hp):
    s = hp.build_hyperbolic(2, 10)
    assert (2, 2) in s and (4, 3) not in s
    with pytest.raises(KeyError):
        s.position((4, 3))
    for o in range(s.size):
        assert s.position(s.index_at(o)) == o
    j = (2, 2)
    assert hp.neighbor(s, j, 1, -1) == s.position((1, 2))
    assert hp.neighbor(s, j, 1, +1) is None
    assert hp.neighbor(s, (0, 0), 1, -1) is None
    with pytest.raises(KeyError):
        hp.neighbor(s, (9, 9), 1, 1)
    with pytest.raises(ValueError):
        hp.neighbor(s, j, 1, 2)
    with pytest.raises(ValueError):
        hp.neighbor(s, j, 3, 1)
    f = hp.build_full(2, 3)
    assert f.size == 16 and f.index_at(1) == (0, 1) and f.index_at(15) == (3, 3)
    assert f.position((2, 1)) == 9
    with pytest.raises(ValueError):
        hp.build_full(0, 3)
    with pytest.raises(ValueError):
        hp.build_hyperbolic(2, -1)


def test_slab_sets(hp):
    f = hp.build_full(3, 7)
    sl = hp.build_slab(3, 7, 2, 5)
    assert sl.size == 3 * 64
    assert np.array_equal(sl.indices, f.indices[2 * 64:5 * 64])
    d, u = sl.neighbor_ordinals(1)
    assert (d[:64] == -1).all() and (u[-64:] == -1).all()


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg5", "cfg3"])
def test_full_size_digests(hp, name):
    """Full-size cfg3 (n = 35,920,101) / cfg5 sets vs the reference's own sha256 digests."""
    path = GOLDEN / "digests.json"
    if not path.exists():
        pytest.skip("digests not generated")
    rec = json.loads(path.read_text()).get(name)
    if rec is None:
        pytest.skip(f"no digest for {name}")
    s = hp.build_hyperbolic(rec["dim"], rec["bound"])
    assert s.size == rec["size"]

    def h(t):
        return hashlib.sha256(t.cpu().numpy().astype("<i8").tobytes()).hexdigest()

    assert h(s.indices_device()) == rec["indices"]
    for a in range(1, rec["dim"] + 1):
        d, u = s.neighbor_tables_device(a)
        assert h(d) == rec[f"down{a}"], a
        assert h(u) == rec[f"up{a}"], a
