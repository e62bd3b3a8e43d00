"""Command-line driver (pkg/src/hitdns/cli.py semantics) on the GPU backend.

CPU: configuration parsing, validation, echo round trip and exit codes
(pkg/tests/test_cli.py style).  GPU: init -> run -> spectrum through the CLI;
an exact-mode RK4 run of config 1 reproduces the reference's final state.
"""

import hashlib
import os

import numpy as np
import pytest
import torch

import paper_2211_16718_b200 as hd
from paper_2211_16718_b200 import cli


def test_parse_config_text_and_overrides(tmp_path):
    path = tmp_path / "run.cfg"
    path.write_text("# comment\nn = 32\nscheme = rk4   # trailing\n\ncfl = 0.3\n")
    cfg = cli.load_config(str(path), ["seed=7", "mu=none"])
    assert (cfg.n, cfg.scheme, cfg.cfl, cfg.seed, cfg.mu) == (32, "rk4", 0.3, 7, None)
    # the echo is reparseable and resolves mu from re_lambda
    again = cli.load_config(None, [l.replace(" = ", "=") for l in cli.config_echo(cfg).splitlines()])
    assert again.mu == pytest.approx(hd.viscosity_from_re_lambda(hd.HitParams()), rel=1e-15)
    assert again.n == 32 and again.cfl == 0.3


@pytest.mark.parametrize("sets", [["scheme=rk5"], ["dt=0.1", "cfl=0.2"], ["n=2"], ["nope=1"],
                                  ["n=abc"], ["layout=aos"], ["mode=turbo"], ["bad"]])
def test_config_errors_exit_2(sets, capsys):
    argv = ["run"]
    for s in sets:
        argv += ["--set", s]
    assert cli.main(argv) == 2
    assert "configuration error" in capsys.readouterr().err


def test_missing_files_exit_4(tmp_path, capsys):
    assert cli.main(["spectrum", "--in", str(tmp_path / "missing.bin")]) == 4
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"not a solution file at all, just bytes" * 4)
    assert cli.main(["spectrum", "--in", str(bad)]) == 4


def test_time_params_defaults():
    cfg = cli.load_config(None, [])
    tp = cli.time_params(cfg)
    assert tp.cfl == 0.4 and tp.dt is None
    assert tp.t_final == pytest.approx(3.0 * hd.eddy_turnover_time(hd.HitParams()))


@pytest.mark.gpu
def test_gpu_init_run_spectrum(tmp_path, traj32_golden):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    init = str(tmp_path / "ic.bin")
    assert cli.main(["init", "--set", "n=32", "--out", init]) == 0
    assert os.path.exists(init + ".config")
    out = str(tmp_path / "final.bin")
    sets = ["n=32", "scheme=rk4", "cfl=0.4", "mu=0.006", "max_steps=10", "mode=exact"]
    argv = ["run", "--in", init, "--out", out]
    for s in sets:
        argv += ["--set", s]
    assert cli.main(argv) == 0
    fields, t = hd.read_solution(out)
    body = fields.interior().cpu().numpy()
    assert hashlib.sha256(np.ascontiguousarray(body).tobytes()).hexdigest() == traj32_golden["final_sha256"]
    assert t == traj32_golden["t"]
    with open(out + ".log") as fh:
        assert len([l for l in fh if l.strip() and not l.startswith("#")]) >= 10
    assert cli.main(["spectrum", "--in", out]) == 0
    ks, es = hd.read_spectrum(out + ".spectrum.txt")
    assert list(ks) == list(range(1, 16))
    it = fields.interior()
    table = hd.compute_spectrum(it[1] / it[0], it[2] / it[0], it[3] / it[0])
    assert np.allclose(es, np.array([e for _, e in table.rows()]), rtol=1e-12, atol=0.0)
    assert table.total() == pytest.approx(traj32_golden["ke"][-1], rel=1e-9)
