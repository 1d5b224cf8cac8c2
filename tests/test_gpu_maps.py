"""restrict / extend / reduction_error / reduction_local_mask on the device and the device CLI,
against the REFERENCE's outputs (tests/golden/maps.npz from tests/golden/make_golden_maps.py;
error_lab.py:114-148, index_set.py:296-319, cli.py:188-217 and 299-314) and against the
reference's own CLI properties (tests/test_cli.py:96-116: byte-identical reruns, --jobs only
changes its header line)."""

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLDEN / "maps.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="module")
def hp():
    import paper_1403_3511_b200 as hp

    return hp


def _cases(gold):
    for k in gold:
        if k.startswith("red_") and k.endswith("_comp"):
            _, pot, dim, bound, deg, beta, _ = k.split("_")
            yield k[:-5], pot, int(dim), int(bound), int(deg), int(beta)


def test_reduction_error_matches_reference(hp, gold):
    for key, pot, dim, bound, deg, beta in _cases(gold):
        s = hp.build_hyperbolic(dim, bound)
        ap = hp.interpolate(hp.potential_by_name(pot, dim), deg)
        rep = hp.reduction_error(s, ap, hp.make_decay_vector(s, beta))
        ref = gold[key + "_comp"]
        # components are |difference| of two matvecs that agree to ~1e-16 relative: compare on
        # the scale of the vectors, and the large components relatively
        assert np.max(np.abs(rep.components - ref)) <= 1e-12 * max(1.0, float(np.max(ref)))
        assert rep.max_norm == pytest.approx(float(gold[key + "_max"]), rel=1e-10, abs=1e-15)
        mask = hp.reduction_local_mask(s, ap)
        assert np.array_equal(mask, gold[key + "_mask"])
        if mask.any():
            assert float(np.max(rep.components[mask])) < 1e-13


def test_reduction_error_device_tensors(hp):
    import torch

    s = hp.build_hyperbolic(3, 10)
    ap = hp.interpolate(hp.potential_by_name("henon-heiles", 3), 3)
    v = hp.make_decay_vector(s, 2)
    host = hp.reduction_error(s, ap, v)
    dev = hp.reduction_error(s, ap, hp.CoeffVector(s, torch.from_numpy(v.data).cuda()))
    assert dev.components.is_cuda
    assert np.array_equal(dev.components.cpu().numpy(), host.components)
    assert dev.metadata["measure"] == "reduction" and dev.metadata["full_size"] == 11 ** 3


def test_full_cube_has_no_reduction_error(hp):
    s = hp.build_full(2, 9)
    ap = hp.interpolate(hp.potential_by_name("torsional", 2), 4)
    rep = hp.reduction_error(s, ap, hp.make_decay_vector(s, 3))
    assert rep.max_norm == 0.0


def test_restrict_extend_batched_and_real(hp):
    import torch

    full, sub = hp.build_full(4, 5), hp.build_hyperbolic(4, 5)
    X = torch.randn(3, full.size, dtype=torch.float64, device="cuda")
    pos = torch.from_numpy(sub.indices @ (6 ** np.arange(3, -1, -1))).cuda()
    R = hp.restrict(hp.CoeffVector(full, X[1]), sub).data
    assert torch.equal(R, X[1][pos])
    from paper_1403_3511_b200.index_set import _map_call

    RB = _map_call("restrict", sub, full, X)
    assert torch.equal(RB, X[:, pos])
    EB = _map_call("extend", sub, full, RB)
    assert torch.equal(EB[:, pos], RB) and float(EB.abs().sum()) == pytest.approx(float(RB.abs().sum()))


def _parse(text):
    head, cols, rows = {}, None, []
    for ln in text.splitlines():
        if ln.startswith("# "):
            k, _, v = ln[2:].partition("=")
            head[k] = v
        elif cols is None:
            cols = ln.split(",")
        else:
            rows.append(ln.split(","))
    return head, cols, rows


def test_cli_rederr_matches_reference_csv(gold, capsys):
    from paper_1403_3511_b200.cli import main

    for i in range(2):
        argv = [str(a) for a in gold[f"cli{i}_argv"]]
        assert main(argv) == 0
        mine = _parse(capsys.readouterr().out)
        ref = _parse(str(gold[f"cli{i}_text"]))
        assert mine[1] == ref[1]
        assert {k: v for k, v in mine[0].items() if k != "backend"} == ref[0]
        assert len(mine[2]) == len(ref[2])
        for a, b in zip(mine[2], ref[2]):
            assert a[:3] == b[:3]
            for x, y in zip(a[3:], b[3:]):
                assert float(x) == pytest.approx(float(y), rel=1e-9, abs=1e-14)


def test_cli_reruns_byte_identical_and_jobs_header_only(tmp_path, capsys):
    from paper_1403_3511_b200.cli import main

    base = ["rederr", "--kmax", "8,12", "--degree", "4", "--beta", "3"]
    a, b, c = tmp_path / "a.csv", tmp_path / "b.csv", tmp_path / "c.csv"
    assert main(base + ["--out", str(a)]) == 0
    assert main(base + ["--out", str(b)]) == 0
    assert main(base + ["--jobs", "2", "--out", str(c)]) == 0
    capsys.readouterr()
    assert a.read_bytes() == b.read_bytes() and b"\r" not in a.read_bytes()
    strip = lambda p: [ln for ln in p.read_text().splitlines() if not ln.startswith("# jobs=")]  # noqa: E731
    assert strip(a) == strip(c) and "# jobs=2" in c.read_text()


def test_cli_bench_and_propagate(capsys):
    from paper_1403_3511_b200.cli import main

    assert main(["bench", "--kmax", "6,8", "--degree", "3"]) == 0
    head, cols, rows = _parse(capsys.readouterr().out)
    assert cols == ["dim", "bound", "set_size", "nterms", "t_fast_s", "t_dense_s", "ratio", "dense_status"]
    assert "dense_cap" in head and all(float(r[4]) > 0 and r[-1] == "skipped_no_dense" for r in rows)
    assert main(["propagate", "--kmax", "6", "--degree", "3", "--h", "1/2,1/4", "--lanczos", "4",
                 "--reference-steps", "64", "--reference-lanczos", "8"]) == 0
    head, cols, rows = _parse(capsys.readouterr().out)
    assert head["scheme"] == "midpoint" and head["reference"] == "fast-gl2"
    assert [r[5] for r in rows] == ["1/2", "1/4"]
    e = [float(r[7]) for r in rows]
    assert e[0] > e[1] > 0.0   # second order: halving h shrinks the endpoint error


def test_unsorted_custom_set_keeps_the_callers_order(hp):
    """An explicit index list in non-lexicographic order (index_set.py:46-65 keeps the caller's
    row order): every result equals the canonical set's result in that order."""
    import torch

    can = hp.build_hyperbolic(3, 10)
    perm = np.random.default_rng(5).permutation(can.size)
    rows = can.indices[perm]
    s = hp.IndexSet(3, 10, "custom", rows)
    assert s.permuted and np.array_equal(s.indices, rows)
    for i in (0, 7, s.size - 1):
        assert s.position(tuple(rows[i])) == i
    for a in (1, 2, 3):
        d_c, u_c = can.neighbor_ordinals(a)
        d, u = s.neighbor_ordinals(a)
        inv = np.argsort(perm)  # canonical ordinal -> caller row
        assert np.array_equal(d, np.where(d_c[perm] >= 0, inv[np.maximum(d_c[perm], 0)], -1))
        assert np.array_equal(u, np.where(u_c[perm] >= 0, inv[np.maximum(u_c[perm], 0)], -1))
    rng = np.random.default_rng(6)
    v = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
    vc = np.empty_like(v)
    vc[perm] = v
    ap = hp.interpolate(hp.potential_by_name("henon-heiles", 3), 3, 0.2)
    for ref_order in (False, True):
        got = hp.get_applier(s).apply_polynomial(ap, v, ref_order=ref_order)
        want = hp.get_applier(can).apply_polynomial(ap, vc, ref_order=ref_order)[perm]
        assert np.array_equal(got, want) if ref_order else rel_l2(got, want) <= 1e-14
    assert np.array_equal(hp.get_applier(s).apply_coordinate(2, v), hp.get_applier(can).apply_coordinate(2, vc)[perm])
    full = hp.build_full(3, 10)
    e = hp.extend(hp.CoeffVector(s, v), full)
    assert np.array_equal(e.data, hp.extend(hp.CoeffVector(can, vc), full).data)
    assert np.array_equal(hp.restrict(e, s).data, v)
    rep = hp.reduction_error(s, ap, hp.CoeffVector(s, v))
    rep_c = hp.reduction_error(can, ap, hp.CoeffVector(can, vc))
    assert np.allclose(rep.components, rep_c.components[perm], rtol=0, atol=1e-14)
    assert np.array_equal(hp.reduction_local_mask(s, ap), hp.reduction_local_mask(can, ap)[perm])
    spec = hp.potential_by_name("henon-heiles", 3)
    fu, fc = hp.FastHamiltonian(s, spec, 3), hp.FastHamiltonian(can, spec, 3)
    sch = hp.MagnusScheme.from_name("midpoint")
    yu = hp.propagate_magnus(sch, fu.matvec_at, v, 0.0, 0.05, 5, 6)
    yc = hp.propagate_magnus(sch, fc.matvec_at, vc, 0.0, 0.05, 5, 6)
    assert rel_l2(yu, yc[perm]) <= 1e-13
    y1, fac = hp.magnus_step(sch, fu.matvec_at, v, 0.0, 0.01, 6)
    y1c, facc = hp.magnus_step(sch, fc.matvec_at, vc, 0.0, 0.01, 6)
    assert rel_l2(y1, y1c[perm]) <= 1e-13 and np.allclose(fac.alpha, facc.alpha, rtol=1e-13)
    assert rel_l2(fac.basis, facc.basis[perm]) <= 1e-13
    # a pinned host tensor comes back as a host tensor
    yt = fu.propagate(sch, torch.from_numpy(v).pin_memory(), 0.0, 0.01, 2, 6)
    assert not yt.is_cuda and rel_l2(yt.numpy(), fc.propagate(sch, vc, 0.0, 0.01, 2, 6)[perm]) <= 1e-13


def test_decay_vector_matches_reference(hp, gold):
    import torch

    for key in [k for k in gold if k.startswith("decay_")]:
        _, kind, dim, bound, beta, norm = key.split("_")
        s = (hp.build_hyperbolic if kind == "hyperbolic" else hp.build_full)(int(dim), int(bound))
        v = hp.make_decay_vector(s, int(beta), normalized=bool(int(norm)))
        assert isinstance(v.data, np.ndarray)
        assert np.max(np.abs(v.data - gold[key])) <= 1e-15 * np.max(np.abs(gold[key]))
        d = hp.make_decay_vector(s, int(beta), normalized=bool(int(norm)), device=True)
        assert d.data.is_cuda and torch.equal(d.data.cpu(), torch.from_numpy(v.data))
    with pytest.raises(ValueError, match="positive integer"):
        hp.make_decay_vector(hp.build_full(2, 3), 0)
