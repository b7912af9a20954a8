"""The LIBSVM-style CLI end to end on the GPU: data file -> plssvm train ->
model file -> plssvm predict -> labels, checked against the oracle (training, Eq. 11-16) and
the oracle's LIBSVM format readers.  Examples from SPEC.md's cli module."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import paper_2202_12674_b200 as pl
import synth
from oracle import libsvm_io as ref

pytestmark = pytest.mark.gpu


def _cli(*args):
    r = subprocess.run([pl.cli_path(), *map(str, args)], capture_output=True, text=True, timeout=300)
    return r


def test_cli_spec_3point_example(tmp_path):
    """S:475 `train -t 0 -c 1 -e 1e-12 tiny3` -> rho -5/3 +- 1e-10; S:483 predict -> 100% (3/3)."""
    data = tmp_path / "tiny3.libsvm"
    data.write_text("+1 1:1\n+1 1:2\n-1 1:3\n")
    r = _cli("train", "-t", 0, "-c", 1, "-e", 1e-12, data)
    assert r.returncode == 0, r.stderr
    assert "CG iterations" in r.stdout and "| cg " in r.stdout and "| total " in r.stdout
    M = ref.parse_model((tmp_path / "tiny3.libsvm.model").read_text())
    assert abs(-M["b"] - (-5 / 3)) <= 1e-10
    assert np.allclose(sorted(M["alpha"]), sorted([0.0, 2 / 3, -2 / 3]), atol=1e-10)
    r = _cli("predict", data, tmp_path / "tiny3.libsvm.model", tmp_path / "out")
    assert r.returncode == 0, r.stderr
    assert "Accuracy = 100% (3/3)" in r.stdout
    assert (tmp_path / "out").read_text().split() == ["1", "1", "-1"]


def test_cli_label_map_0_1(tmp_path):
    """labels {0, 1} with 0 first -> 0 is the +1 class; predictions are emitted as 0 / 1."""
    X, y, Z, yz = synth.planes(300, 6, 100, seed=12)
    y01 = np.where(y > 0, 0.0, 1.0)
    if y01[0] != 0.0:
        y01 = 1.0 - y01
    ref_text = ref.write_libsvm(X, y01)
    (tmp_path / "tr").write_text(ref_text)
    (tmp_path / "te").write_text(ref.write_libsvm(Z, np.where(yz > 0, y01[0], 1.0 - y01[0])))
    assert _cli("train", "-t", 2, "-e", 1e-10, tmp_path / "tr", tmp_path / "m").returncode == 0
    M = ref.parse_model((tmp_path / "m").read_text())
    assert M["labels"] == [0.0, 1.0]
    r = _cli("predict", tmp_path / "te", tmp_path / "m", tmp_path / "out")
    assert r.returncode == 0, r.stderr
    assert set((tmp_path / "out").read_text().split()) <= {"0", "1"}


@pytest.mark.parametrize("kernel,extra", [(2, []), (1, ["-d", 3, "-r", 1.0]), (0, [])])
def test_cli_model_matches_oracle_training(tmp_path, kernel, extra):
    X, y, Z, yz = synth.planes(600, 17, 200, seed=30 + kernel)
    (tmp_path / "tr").write_text(ref.write_libsvm(X, y))
    (tmp_path / "te").write_text(ref.write_libsvm(Z, yz))
    r = _cli("train", "-t", kernel, "-e", 1e-10, *extra, tmp_path / "tr", tmp_path / "m")
    assert r.returncode == 0, r.stderr
    M = ref.parse_model((tmp_path / "m").read_text())
    gamma = 1.0 / 17  # CLI default 1/num_features
    assert M["gamma"] == (gamma if kernel else 0.0)
    degree, coef0 = (3, 1.0) if kernel == 1 else (3, 0.0)
    a_ref, b_ref, _, _ = oracle.train(X, y, kernel, gamma, degree, coef0, 1.0, 1e-10)
    # model SV order: y = +1 points first (LIBSVM class grouping), each group in input order
    order = np.r_[np.where(y == y[0])[0], np.where(y != y[0])[0]]
    a_ref = a_ref[order] if y[0] == 1.0 else -a_ref[order]  # first-seen label is the +1 class
    b_exp = b_ref if y[0] == 1.0 else -b_ref
    assert np.linalg.norm(M["alpha"] - a_ref) <= 1e-7 * np.linalg.norm(a_ref)
    assert abs(M["b"] - b_exp) <= 1e-7 * max(abs(b_exp), np.abs(a_ref).max())
    r = _cli("predict", tmp_path / "te", tmp_path / "m", tmp_path / "out")
    assert r.returncode == 0, r.stderr
    _, lab_ref = oracle.predict(X, *oracle.train(X, y, kernel, gamma, degree, coef0, 1.0, 1e-10)[:2], Z, kernel,
                                gamma, degree, coef0)
    got = np.array([float(v) for v in (tmp_path / "out").read_text().split()])
    assert np.array_equal(got, lab_ref.astype(np.float64))
    acc = float(r.stdout.split("Accuracy = ")[1].split("%")[0])
    assert abs(acc - 100.0 * np.mean(lab_ref == yz)) < 1e-2


def test_cli_fp32_and_scaled_workflow(tmp_path):
    """svm-scale -> train -> predict with the test file restored to the training ranges."""
    X, y, Z, yz = synth.planes(400, 12, 150, seed=8)
    (tmp_path / "tr").write_text(ref.write_libsvm(X * 5 + 2, y))
    (tmp_path / "te").write_text(ref.write_libsvm(Z * 5 + 2, yz))
    r = _cli("scale", "-s", tmp_path / "range", tmp_path / "tr")
    assert r.returncode == 0
    (tmp_path / "tr.s").write_text(r.stdout)
    r = _cli("scale", "-r", tmp_path / "range", tmp_path / "te")
    assert r.returncode == 0
    (tmp_path / "te.s").write_text(r.stdout)
    assert _cli("train", "--fp32", "-e", 1e-6, tmp_path / "tr.s", tmp_path / "m").returncode == 0
    r = _cli("predict", tmp_path / "te.s", tmp_path / "m", tmp_path / "out")
    assert r.returncode == 0
    assert float(r.stdout.split("Accuracy = ")[1].split("%")[0]) > 80.0
