"""Wire formats, run reports, CLI exit codes and the multi-shift driver.

CPU tests pin the SBM reader/writer against the reference's own code (oracle/_ref:
banded.hpp:115-154) and check the exit
codes that need no device (tools/specproj.cpp:33-36).  GPU tests run the CLI's
project / verify and the multi-shift driver end to end.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_1608_01164_b200 as S
from oracle import ref as R

CLI = S.cli_path()
need_cli = pytest.mark.skipif(not os.path.exists(CLI), reason="CLI not built (run __graft_entry__.build())")
need_ref = pytest.mark.skipif(not R.ref_available(), reason="reference build (oracle/_ref) not available")


def _cli(*args, timeout=600):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=timeout)


def test_sbm_roundtrip(tmp_path):
    A = S.random_banded(37, 4, 5)
    p = str(tmp_path / "a.sbm")
    S.write_sbm(p, A)
    B = S.read_sbm(p)
    assert (B.n, B.b) == (37, 4)
    for d in range(5):
        np.testing.assert_array_equal(A.bands[d], B.bands[d])
    with open(p) as f:
        assert f.readline().strip() == "SBM 37 4"


def test_sbm_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.sbm"
    p.write_text("SBX 4 1\n1 2 3 4\n1 2 3\n")
    with pytest.raises(ValueError):
        S.read_sbm(str(p))
    p.write_text("SBM 4 1\n1 2 3 4\n1 2\n")
    with pytest.raises(ValueError):
        S.read_sbm(str(p))
    p.write_text("SBM 4 1\n1 2 nan 4\n1 2 3\n")
    with pytest.raises(ValueError):
        S.read_sbm(str(p))


@need_ref
def test_sbm_matches_reference_writer_and_reader(tmp_path):
    ref = R.RefLib()
    A = S.dimer_chain(101, 1.0, 0.37, 0.1, 3, b=3, s=1e-3)
    ours, theirs = str(tmp_path / "ours.sbm"), str(tmp_path / "theirs.sbm")
    S.write_sbm(ours, A)
    ref.write_sbm(theirs, A.bands)
    assert open(ours).read() == open(theirs).read()          # byte-identical text
    back = ref.read_sbm(ours)
    for d in range(4):
        np.testing.assert_array_equal(back[d], A.bands[d])


@need_cli
def test_cli_exit_codes(tmp_path):
    assert _cli().returncode == 2                                     # no subcommand
    assert _cli("project").returncode == 2                            # --in required
    assert _cli("project", "--in", "x", "--bogus", "1").returncode == 2
    assert _cli("project", "--in", str(tmp_path / "missing.sbm")).returncode == 3
    assert _cli("generate", "--n", "8", "--band", "9", "--out", str(tmp_path / "z.sbm")).returncode == 2  # not built
    assert _cli("bench", "--sizes", "8", "--band", "9").returncode == 2
    A = S.random_banded(64, 2, 1)
    p = str(tmp_path / "a.sbm")
    S.write_sbm(p, A)
    r = _cli("verify", "--in", p, "--oracle-cap", "32")
    assert r.returncode == 5 and "oracle cap" in r.stderr


# ------------------------------------------------------------------ GPU
@need_cli
@pytest.mark.gpu
def test_cli_project_report(tmp_path):
    A = S.dimer_chain(2048, 1.0, 0.5, 0.1, 1)
    p, rep = str(tmp_path / "pr1.sbm"), str(tmp_path / "rep.json")
    S.write_sbm(p, A)
    r = _cli("project", "--in", p, "--nmin", "128", "--report", rep)
    assert r.returncode == 0, r.stderr
    d = json.load(open(rep))
    assert list(d) == ["input", "params", "iterations", "per_iteration", "errors", "totals"]
    assert d["input"] == {"file": p, "n": 2048, "b": 1, "gap": None, "seed": None}
    assert d["errors"] is None
    direct = S.hqdwh(S.read_sbm(p), 128, 1e-10)
    assert d["iterations"] == direct.iterations
    assert d["params"]["alpha"] == direct.alpha and d["params"]["l0"] == direct.l0
    assert round(d["totals"]["trace_p"]) == 1024 and abs(d["totals"]["trace_p"] - 1024) < 1e-8
    assert [x["k"] for x in d["per_iteration"]] == list(range(1, direct.iterations + 1))
    mine = S.run_report(p, S.read_sbm(p), 128, 1e-10, 1e-15, 0.0, direct, d["totals"]["wall_ms"])
    assert list(mine) == list(d) and mine["totals"]["max_rank"] == d["totals"]["max_rank"]


@need_cli
@pytest.mark.gpu
def test_cli_verify_errors(tmp_path):
    A = S.dimer_chain(512, 1.0, 0.6, 0.1, 4)
    p = str(tmp_path / "v.sbm")
    S.write_sbm(p, A)
    r = _cli("verify", "--in", p, "--nmin", "64")
    assert r.returncode == 0, r.stderr
    e = json.loads(r.stdout)["errors"]
    assert e["e_id"] < 1e-8 and e["e_trace"] < 1e-8 and e["e_sp"] < 1e-8, e


@need_cli
@pytest.mark.gpu
def test_cli_cholesky_breakdown_exit_4(tmp_path):
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "npd_case.npz"))
    A = S.BandedSymmetric.from_packed(int(g["n"]), int(g["b"]), g["bands"])
    p = str(tmp_path / "npd.sbm")
    S.write_sbm(p, A)
    r = _cli("project", "--in", p, "--nmin", str(int(g["n_min"])), "--eps", repr(float(g["eps"])))
    assert r.returncode == 4, (r.returncode, r.stderr)


@pytest.mark.gpu
def test_multi_shift_matches_single_projectors():
    A = S.dimer_chain(1024, 1.0, 0.5, 0.1, 6)
    shifts = [0.0, 0.9, -0.9]
    multi = S.hqdwh_shifts(A, shifts, 64, 1e-10, max_concurrent=3)
    ev = np.linalg.eigvalsh(np.diag(A.bands[0]) + np.diag(A.bands[1], 1) + np.diag(A.bands[1], -1))
    X = np.random.default_rng(1).standard_normal((A.n, 4))
    for mu, r in zip(shifts, multi):
        single = S.hqdwh(A.shifted(mu), 64, 1e-10)
        assert r.iterations == single.iterations
        # concurrency does not change the arithmetic; run to run the default path agrees to the
        # truncation level (Races), so compare the operators, not the bits
        assert np.abs(r.apply(X) - single.apply(X)).max() <= 1e-9
        assert round(r.P.trace()) == int((ev < mu).sum())


@pytest.mark.gpu
def test_multi_shift_over_devices():
    """spg_hqdwh_shifts_devices on the visible GPUs (one here): same results as single calls,
    device bookkeeping, result calls from a thread whose current device differs are safe."""
    A = S.dimer_chain(1024, 1.0, 0.5, 0.1, 6)
    shifts = [0.0, 0.9, -0.9, 0.3]
    rs, dev_of = S.hqdwh_shifts_devices(A, shifts, 64, 1e-10)              # every visible device
    assert all(d >= 0 for d in dev_of)
    X = np.random.default_rng(1).standard_normal((A.n, 4))
    L = S.load_library()
    for mu, r, d in zip(shifts, rs, dev_of):
        assert L.spg_result_device(r._handle) == d
        single = S.hqdwh(A.shifted(mu), 64, 1e-10)
        assert np.abs(r.apply(X) - single.apply(X)).max() <= 1e-9
    rs1, dev1 = S.hqdwh_shifts_devices(A, shifts[:2], 64, 1e-10, devices=[0], per_device_concurrent=1)
    assert dev1 == [0, 0]
    assert np.abs(rs1[1].apply(X) - rs[1].apply(X)).max() <= 1e-9
    with pytest.raises(ValueError):
        S.hqdwh_shifts_devices(A, shifts, 64, 1e-10, devices=[0, 99])
    with pytest.raises(ValueError):
        S.hqdwh_shifts_devices(A, shifts, 64, 1e-10, devices=[0, 0])


@need_cli
@pytest.mark.gpu
def test_cli_multi_shift_reports(tmp_path):
    A = S.dimer_chain(512, 1.0, 0.5, 0.1, 2)
    p = str(tmp_path / "m.sbm")
    S.write_sbm(p, A)
    r = _cli("project", "--in", p, "--nmin", "64", "--shifts", "0,0.9")
    assert r.returncode == 0, r.stderr
    reps = json.loads(r.stdout)
    assert [x["params"]["shift"] for x in reps] == [0.0, 0.9]
    ev = np.linalg.eigvalsh(np.diag(A.bands[0]) + np.diag(A.bands[1], 1) + np.diag(A.bands[1], -1))
    assert [round(x["totals"]["trace_p"]) for x in reps] == [int((ev < 0).sum()), int((ev < 0.9).sum())]
