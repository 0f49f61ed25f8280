"""CLI routing of the hot-path subcommands (reference cli.py).

The golden files tests/golden/cli_* are the reference CLI's own outputs for
the wind-scale pipeline of pkg/tests/test_cli.py:14-40 (make_golden.py).  Our
``fit``/``div`` outputs must be byte-identical (the fp64 paths are bitwise and
the files store fp32); ``gradmag`` within one fp32 ulp (GPU hypot is within
an ulp of glibc's); ``lcp`` CSV cells within the fp64 tail tolerance 1e-12.
Exit-code and argument-error cases run on the CPU (no kernel is reached).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN

gpu = pytest.mark.gpu


def G(name):
    return os.path.join(GOLDEN, f"cli_{name}")


@pytest.fixture(scope="module")
def cli():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2510_01190_b200 import cli

    return cli


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(cli, *argv):
    return cli.cli_main([str(a) for a in argv])


def _payload(path):
    raw = open(path, "rb").read()
    return raw[: raw.index(b"\n") + 1], np.frombuffer(raw[raw.index(b"\n") + 1:], dtype="<f4")


@gpu
def test_fit_div_byte_identical_to_reference(cli, cuda, tmp_path):
    mu, sg, dmu, dsg = (tmp_path / f for f in ("mu.duq", "sg.duq", "dmu.duq", "dsg.duq"))
    assert run(cli, "fit", "--in", G("wind.duq"), "--out-mu", mu, "--out-sigma", sg) == 0
    assert mu.read_bytes() == open(G("mu.duq"), "rb").read()
    assert sg.read_bytes() == open(G("sg.duq"), "rb").read()
    assert run(cli, "div", "--in-mu", mu, "--in-sigma", sg, "--out-mu", dmu, "--out-sigma", dsg) == 0
    assert dmu.read_bytes() == open(G("dmu.duq"), "rb").read()
    assert dsg.read_bytes() == open(G("dsg.duq"), "rb").read()


@gpu
def test_lcp_csv_matches_reference(cli, cuda, tmp_path):
    out = tmp_path / "lcp.csv"
    assert run(cli, "lcp", "--in-mu", G("dmu.duq"), "--in-sigma", G("dsg.duq"), "--iso", "-2.525",
               "--out", out) == 0
    got = out.read_text().splitlines()
    ref = open(G("lcp.csv")).read().splitlines()
    assert got[0] == ref[0] == "cell_i,cell_j,probability"
    assert len(got) == len(ref) == 1 + 23 * 23
    for a, b in zip(got[1:], ref[1:]):
        ia, ja, pa = a.split(",")
        ib, jb, pb = b.split(",")
        assert (ia, ja) == (ib, jb)
        assert abs(float(pa) - float(pb)) <= 1e-12 * max(1e-300, abs(float(pb))) + 1e-15


@gpu
def test_gradmag_matches_reference(cli, cuda, tmp_path):
    out = tmp_path / "gm.duq"
    assert run(cli, "gradmag", "--in", G("wind.duq"), "--out", out) == 0
    h1, got = _payload(out)
    h2, ref = _payload(G("gm.duq"))
    assert h1 == h2
    ulp = np.spacing(np.abs(ref).astype(np.float32))
    assert np.all(np.abs(got - ref) <= ulp)


@gpu
def test_mc_with_metrics(cli, cuda, tmp_path):
    metrics = tmp_path / "metrics.csv"
    assert run(cli, "mc", "--in-mu", G("mu.duq"), "--in-sigma", G("sg.duq"), "--samples", 500,
               "--seed", 4, "--out-mean", tmp_path / "m.duq", "--out-std", tmp_path / "s.duq",
               "--sse-against", G("dmu.duq"), G("dsg.duq"), "--metrics-out", metrics) == 0
    rows = dict(line.split(",") for line in metrics.read_text().splitlines()[1:])
    assert float(rows["e_m"]) < 0.1
    assert float(rows["sse"]) >= 0.0


@gpu
def test_bench_csv(cli, cuda, tmp_path, capsys):
    csv = tmp_path / "bench.csv"
    assert run(cli, "bench", "--in", G("wind.duq"), "--samples-list", "100", "--threads-list", "2",
               "--runs", "2", "--out-csv", csv) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == "label,runs,mean_s,min_s,max_s,sse,speedup_vs_analytic_serial"
    assert [line.split(",")[0] for line in lines[1:]] == ["analytic_serial", "analytic_threads_2", "mc_100"]
    assert float(lines[3].split(",")[5]) > 0


def test_exit_codes(cli, tmp_path, capsys):
    assert run(cli, "no-such-command") == 1
    assert run(cli, "fit", "--in", tmp_path / "missing.duq", "--out-mu", "a", "--out-sigma", "b") == 2
    bad = tmp_path / "bad.duq"
    bad.write_bytes(b"BOGUS\n")
    assert run(cli, "fit", "--in", bad, "--out-mu", "a", "--out-sigma", "b") == 2
    one = tmp_path / "one.duq"
    one.write_bytes(b"DIVUQ1 2 2 1 1 1\n" + b"\x00" * 32)
    assert run(cli, "fit", "--in", one, "--out-mu", "a", "--out-sigma", "b") == 2  # DataError
    assert run(cli, "div", "--in-mu", G("mu.duq"), "--in-sigma", G("wind.duq"),
               "--out-mu", "a", "--out-sigma", "b") == 2  # model files need one block
    assert run(cli, "fit", "--in", G("wind.duq")) == 1  # missing required flags
    assert run(cli, "--help") == 0
    assert "error" in capsys.readouterr().err


@pytest.mark.parametrize("cmd", ["gen", "contour", "render", "validate-1d"])
def test_out_of_scope_subcommands_are_usage_errors(cli, cmd, capsys):
    assert run(cli, cmd, "--anything") == 1
    assert "reference CLI" in capsys.readouterr().err


def test_lcp_ppm_output_is_a_usage_error(cli, tmp_path, capsys):
    assert run(cli, "lcp", "--in-mu", G("dmu.duq"), "--in-sigma", G("dsg.duq"), "--iso", "0",
               "--out", tmp_path / "x.csv", "--out", tmp_path / "x.ppm") == 1
    assert not (tmp_path / "x.csv").exists()


def test_csv_helpers(tmp_path):
    from paper_2510_01190_b200 import io as dio

    assert dio.csv_float(0.1) == "0.1" and dio.csv_float(1) == "1.0"
    p = tmp_path / "t.csv"
    dio.write_csv(p, "a,b", [(1, "x"), (2, dio.csv_float(1e-300))])
    assert p.read_bytes() == b"a,b\n1,x\n2,1e-300\n"
