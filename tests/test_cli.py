"""Drop-in `nonloc` CLI (§8(f) row 2; reference tools/nonloc_main.cpp,
src/config.cpp, src/bench.cpp): CSV layout, '# config:' line, %.17g values,
slope lines and exit codes 0/1/2, against the compiled reference's numbers
(golden fixtures). Parsing, config files and `split` run on the CPU; apply /
bench / solve need the B200."""
import io
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden

EXE = os.path.join(ROOT, "paper_1905_08375_b200", "_lib", "nonloc")


@pytest.fixture(scope="module")
def cli():
    from paper_1905_08375_b200 import build
    build.build()
    assert os.path.exists(EXE)
    return EXE


def run(args, **kw):
    return subprocess.run([EXE] + args, capture_output=True, text=True, timeout=600, **kw)


def csv_rows(text):
    lines = [l for l in text.splitlines() if l and not l.startswith("#")]
    hdr = lines[0].split(",")
    return hdr, [l.split(",") for l in lines[1:]]


def test_usage_errors_exit_1(cli):
    assert run(["--help"]).returncode == 0
    assert run([]).returncode == 1
    assert run(["frobnicate"]).returncode == 1
    assert run(["apply", "--bogus", "1"]).returncode == 1
    assert run(["apply", "--n"]).returncode == 1
    assert run(["apply", "--n", "abc"]).returncode == 1
    assert run(["bench", "--sweep", "8,16"]).returncode == 1          # needs >= 4 sizes
    assert run(["apply", "--sweep", "8,16,32,64"]).returncode == 1    # bench-only flag
    assert run(["rank-profile"]).returncode == 1                       # HODLR: out of scope


def test_split_report(cli):
    from paper_1905_08375_b200 import nonloc as N
    r = run(["split", "--K", "2"])
    assert r.returncode == 0
    first = r.stdout.splitlines()[0]
    assert first.startswith("# config: command=split dim=1 n=256 delta0=0.25 horizon=constant profile=inverse_s")
    assert " split_K=2 " in first and " epsilon=1e-08 tol=1e-10 seed=1" in first
    hdr, rows = csv_rows(r.stdout)
    assert hdr == ["s", "gamma", "p", "kappa"] and len(rows) == 101
    assert rows[0][1] == "inf" and rows[0][3] == "inf"
    sk = N.split(N.RadialProfile.inverse_s(), 2)
    p = N.match_polynomial(2)
    for row in rows[1:-1]:
        s = float(row[0])
        assert float(row[2]) == pytest.approx(np.polyval(p[::-1], s * s), rel=1e-15, abs=1e-15)
        assert float(row[1]) == 1.0 / s
    assert "35/16" not in r.stderr and "s^0:" in r.stderr


def test_config_file_defaults_and_overrides(cli, tmp_path):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("# comment\n\nK = 1\nn=512\ndelta0=0.125\nhorizon=gaussian_bump\n")
    r = run(["--config", str(cfg), "split"])
    assert r.returncode == 0 and " n=512 delta0=0.125 horizon=gaussian_bump " in r.stdout and " split_K=1 " in r.stdout
    r = run(["split", "--config", str(cfg), "--K", "3"])            # explicit flag wins
    assert " split_K=3 " in r.stdout
    bad = tmp_path / "bad.cfg"
    bad.write_text("n=8\nwhat=1\n")
    r = run(["--config", str(bad), "split"])
    assert r.returncode == 1 and "bad.cfg:2: unknown key 'what'" in r.stderr
    out = tmp_path / "o.csv"
    assert run(["split", "--out", str(out)]).returncode == 0 and out.read_text().startswith("# config:")


@pytest.mark.gpu
@pytest.mark.parametrize("name,args", [
    ("trunc_2d_n64_k0", ["--dim", "2", "--n", "64", "--delta0", "0.5", "--seed", "42"]),
    ("trunc_3d_n8_k0", ["--dim", "3", "--n", "8", "--delta0", "0.5", "--seed", "44"]),
    ("trunc_1d_n2048_k3_bump", ["--dim", "1", "--n", "2048", "--K", "3", "--horizon", "gaussian_bump",
                                "--delta0", "0.25", "--seed", "43"]),
])
def test_apply_matches_reference_counters(cli, name, args):
    g = golden(name)
    r = run(["apply"] + args)
    assert r.returncode == 0, r.stderr
    hdr, rows = csv_rows(r.stdout)
    assert hdr == ["N", "recur_calls", "step2_ops", "step3_ops", "dense_pairs", "max_rel_err_vs_dense"]
    N_, rc, s2, s3, pairs, err = rows[0]
    assert [int(N_), int(rc), int(s2), int(s3)] == [int(g["u"].size)] + [int(v) for v in g["counters"]]
    assert int(pairs) == int(g["leaf_pairs"])
    assert float(err) <= 1e-10


@pytest.mark.gpu
def test_bench_sweep_and_slopes(cli):
    r = run(["bench", "--sweep", "256,512,1024,2048", "--delta0", "0.05"])
    assert r.returncode == 0, r.stderr
    hdr, rows = csv_rows(r.stdout)
    assert len(rows) == 4 and hdr[-1] == "max_rel_err_vs_dense"
    slopes = {l.split("=")[0][2:]: float(l.split("=")[1]) for l in r.stdout.splitlines() if l.startswith("# slope_")}
    assert set(slopes) == {"slope_recur_calls", "slope_step23_ops", "slope_dense_pairs", "slope_fast_wall_ns",
                           "slope_dense_wall_ns"}
    assert 1.0 <= slopes["slope_recur_calls"] <= 1.2              # N log N in 1-D (test_tree.cpp:221-233)
    assert 1.9 <= slopes["slope_dense_pairs"] <= 2.1              # fixed delta: pairs ~ N^2


@pytest.mark.gpu
def test_solve_manufactured_cgnr(cli, tmp_path):
    G = golden("solve_dirichlet")
    out = tmp_path / "s.csv"
    r = run(["solve", "--n", "256", "--horizon", "gaussian_bump", "--delta0", "0.25", "--out", str(out)])
    assert r.returncode == 0, r.stderr
    text = out.read_text()
    head = text.split("# solution")[0]
    hdr, rows = csv_rows(head)
    assert hdr == ["method", "N", "iterations", "final_residual", "converged", "manufactured_rel_err"]
    assert rows[0][0] == "CGNR" and rows[0][1] == "256" and rows[0][4] == "1"
    sol = np.array([float(l.split(",")[2]) for l in text.split("index,x,u\n")[1].splitlines()])
    assert np.max(np.abs(sol - G["cgnr_n256_bump_direct"])) <= 1e-6 * np.max(np.abs(G["cgnr_n256_bump_direct"]))
    r = run(["solve", "--n", "128", "--tol", "1e-14", "--max-iter", "2"])
    assert r.returncode == 2                                       # not converged -> conformance exit
