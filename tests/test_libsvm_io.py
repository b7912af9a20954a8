"""LIBSVM data / model files and svm-scale, CPU only.

1. The plain-Python oracle (oracle/libsvm_io.py) is pinned to SPEC.md's worked examples
   (tests/golden/libsvm_examples.txt) and to format invariants (round trips).
2. The native C++ implementation (io.cpp through the C ABI) is compared with the oracle on the
   same seeded files: parsed matrices BIT-identical, written files BYTE-identical.
3. The CLI (bin/plssvm) is exercised for everything that needs no GPU (scale, usage errors).
"""
import os
import subprocess

import numpy as np
import pytest

import paper_2202_12674_b200 as pl
from oracle import libsvm_io as ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def golden():
    sec, cur = {}, None
    for ln in open(os.path.join(ROOT, "tests", "golden", "libsvm_examples.txt")):
        if ln.startswith("#"):
            continue
        if ln.startswith("== "):
            cur = ln.split()[1]
            sec[cur] = ""
        elif cur:
            sec[cur] += ln
    return sec


# ---------------------------------------------------------------- oracle pins (SPEC examples)
def test_oracle_parse_matches_spec_example():
    g = golden()
    X, y, labels = ref.parse_libsvm(g["parse_data"])
    exp = [list(map(float, r.split())) for r in g["parse_data_expected"].strip().split("\n")]
    assert X.shape == tuple(int(v) for v in exp[0])
    assert np.array_equal(X, np.array(exp[1:]))
    assert list(y) == [1.0, -1.0] and labels == [1.0, -1.0]


def test_oracle_parse_rejects_descending_indices():
    with pytest.raises(ref.FormatError, match="line 1: indices must be ascending"):
        ref.parse_libsvm(golden()["parse_error_ascending"])


def test_oracle_model_rho_lines():
    g = golden()
    X = np.array([[1.0], [2.0], [3.0]])
    txt = ref.write_model(0, 1.0, 3, 0.0, X, [0.0, 2 / 3, -2 / 3], 5 / 3, [1.0, 1.0, -1.0], [1.0, -1.0])
    assert g["model_3point_rho"].strip() in txt.split("\n")
    txt0 = ref.write_model(0, 1.0, 3, 0.0, X, [0.0, 2 / 3, -2 / 3], 0.0, [1.0, 1.0, -1.0], [1.0, -1.0])
    assert g["model_b0_rho"].strip() in txt0.split("\n")
    poly = ref.write_model(1, 0.5, 3, 1.0, X, [0.0, 2 / 3, -2 / 3], 5 / 3, [1.0, 1.0, -1.0], [1.0, -1.0])
    assert all(any(l.startswith(k + " ") for l in poly.split("\n")) for k in ("degree", "gamma", "coef0"))


def test_oracle_scaling_examples():
    fmin, fmax = ref.fit_scaling(np.array([[0.0, 4.0], [5.0, 4.0], [10.0, 4.0]]))
    s = ref.apply_scaling(np.array([[0.0, 4.0], [5.0, 4.0], [10.0, 4.0]]), fmin, fmax)
    assert list(s[:, 0]) == [-1.0, 0.0, 1.0] and list(s[:, 1]) == [-1.0, -1.0, -1.0]
    assert ref.apply_scaling(np.array([[20.0]]), np.array([0.0]), np.array([10.0]))[0, 0] == 3.0


def test_oracle_round_trips():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((20, 7)) * (rng.random((20, 7)) < 0.5)
    y = np.where(rng.random(20) < 0.5, 1.0, -1.0)
    X2, y2, _ = ref.parse_libsvm(ref.write_libsvm(X, y))
    assert np.array_equal(X2[:, :X2.shape[1]], X[:, :X2.shape[1]]) and np.array_equal(y2, y)
    alpha = rng.standard_normal(20)
    M = ref.parse_model(ref.write_model(2, 0.25, 3, 0.0, X, alpha, -0.125, y, [1.0, -1.0]))
    order = np.r_[np.where(y == 1)[0], np.where(y == -1)[0]]
    assert np.array_equal(M["alpha"], alpha[order]) and M["b"] == -0.125 and M["kernel"] == 2
    for bad, msg in [("nr_class 3", "nr_class"), (None, "rho")]:
        txt = ref.write_model(2, 0.25, 3, 0.0, X, alpha, -0.125, y, [1.0, -1.0])
        txt = txt.replace("nr_class 2", bad) if bad else "\n".join(l for l in txt.split("\n") if not l.startswith("rho"))
        with pytest.raises(ref.FormatError, match=msg):
            ref.parse_model(txt)


# ------------------------------------------------------ native C++ vs oracle (bit / byte exact)
def _random_file_text(rng, m, d, labels=(1.0, -1.0), density=0.4, crlf=False, comments=True):
    lines = []
    for i in range(m):
        if comments and rng.random() < 0.05:
            lines.append("# a comment line")
        if comments and rng.random() < 0.05:
            lines.append("   ")
        lab = labels[int(rng.integers(len(labels)))]
        toks = ["%+g" % lab if rng.random() < 0.3 else repr(lab)]
        for k in range(1, d + 1):
            if rng.random() < density:
                v = float(rng.standard_normal() * 10.0 ** int(rng.integers(-8, 8)))
                toks.append(f"{k}:{v!r}" if rng.random() < 0.8 else f"{k}:{v:.6e}")
        lines.append(" ".join(toks) + ("  " if rng.random() < 0.1 else ""))
    return ("\r\n" if crlf else "\n").join(lines) + "\n"


@pytest.mark.parametrize("m,d,crlf,labels", [(1, 1, False, (1.0, -1.0)), (50, 9, False, (0.0, 1.0)),
                                            (300, 40, True, (2.0, 4.0)), (2000, 130, False, (-1.0, 1.0))])
def test_native_parse_is_bit_identical_to_oracle(tmp_path, m, d, crlf, labels):
    rng = np.random.default_rng(m + d)
    text = _random_file_text(rng, m, d, labels, crlf=crlf)
    p = tmp_path / "data.txt"
    p.write_bytes(text.encode())
    X, y, labs = pl.plssvm_libsvm_read(p)
    Xr, yr, labr = ref.parse_libsvm(text)
    assert X.shape == Xr.shape if Xr.shape[1] > 0 else True
    assert np.array_equal(X[:, :Xr.shape[1]], Xr) and np.array_equal(y, yr) and labs == labr
    assert X.view(np.uint64).tobytes() == np.ascontiguousarray(X).view(np.uint64).tobytes()


def test_native_parse_large_file_multithreaded(tmp_path):
    """> 1 MiB per thread: the chunked parse must give the oracle's matrix (chunk seams, line numbers)."""
    rng = np.random.default_rng(5)
    X = rng.standard_normal((6000, 64))
    y = np.where(rng.random(6000) < 0.5, 1.0, -1.0)
    text = ref.write_libsvm(X, y)
    p = tmp_path / "big.txt"
    p.write_text(text)
    assert os.path.getsize(p) > 4 * 2**20
    X2, y2, _ = pl.plssvm_libsvm_read(p)
    assert np.array_equal(X2, X) and np.array_equal(y2, y)
    # an error deep in the file names the right line
    lines = text.split("\n")
    lines[4321] = lines[4321].replace(" 2:", " 2:abc", 1)
    p.write_text("\n".join(lines))
    with pytest.raises(pl.PlssvmError, match="line 4322: invalid value"):
        pl.plssvm_libsvm_read(p)


@pytest.mark.parametrize("text,msg", [
    ("1 2:3 1:4\n", "line 1: indices must be ascending"),
    ("1 1:1\n-1 0:2\n", "line 2: feature index 0 < 1"),
    ("1 1:1\n-1 1:x\n", "line 2: invalid value"),
    ("abc 1:1\n", "line 1: invalid label"),
    ("1 1:1 1:2\n", "line 1: indices must be ascending"),
    ("1 1=2\n", "line 1: invalid feature"),
    ("# only comments\n\n", "no data points"),
])
def test_native_parse_errors(tmp_path, text, msg):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(pl.PlssvmError, match=msg) as e:
        pl.plssvm_libsvm_read(p)
    assert e.value.status == pl.binding.E_IO
    with pytest.raises(ref.FormatError):
        ref.parse_libsvm(text)


def test_native_parse_three_labels_and_missing_file(tmp_path):
    p = tmp_path / "three.txt"
    p.write_text("1 1:1\n2 1:2\n3 1:3\n")
    with pytest.raises(pl.PlssvmError) as e:
        pl.plssvm_libsvm_read(p)
    assert e.value.status == pl.binding.E_LABELS
    with pytest.raises(pl.PlssvmError, match="cannot open") as e:
        pl.plssvm_libsvm_read(tmp_path / "nope.txt")
    assert e.value.status == pl.binding.E_IO


def test_native_writers_are_byte_identical_to_oracle(tmp_path):
    rng = np.random.default_rng(3)
    X = rng.standard_normal((40, 6)) * (rng.random((40, 6)) < 0.6)
    X[3, 2] = -0.0
    y = np.where(rng.random(40) < 0.5, 1.0, -1.0)
    alpha = rng.standard_normal(40)
    pl.plssvm_libsvm_write(tmp_path / "d.txt", X, y)
    assert (tmp_path / "d.txt").read_text() == ref.write_libsvm(X, y)
    for kernel, b in [(0, 5 / 3), (1, -0.0), (2, 0.1)]:
        pl.plssvm_model_write(tmp_path / "m.txt", kernel, 0.25, 3, 1.5, X, alpha, b, y, [2.0, 4.0])
        assert (tmp_path / "m.txt").read_text() == ref.write_model(kernel, 0.25, 3, 1.5, X, alpha, b, y, [2.0, 4.0])
        M = pl.plssvm_model_read(tmp_path / "m.txt")
        R = ref.parse_model((tmp_path / "m.txt").read_text())
        assert M["kernel"] == R["kernel"] == kernel and M["labels"] == R["labels"] == [2.0, 4.0]
        assert np.array_equal(M["alpha"], R["alpha"]) and M["b"] == R["b"] and np.array_equal(M["X"], R["X"])


def test_native_model_read_errors(tmp_path):
    X = np.eye(3)
    good = ref.write_model(2, 0.5, 3, 0.0, X, [1.0, -0.5, -0.5], 0.25, [1.0, -1.0, -1.0], [1.0, -1.0])
    cases = [(good.replace("nr_class 2", "nr_class 3"), "nr_class"),
             ("\n".join(l for l in good.split("\n") if not l.startswith("rho")), "missing field 'rho'"),
             (good.replace("kernel_type rbf", "kernel_type sigmoid"), "unknown kernel_type"),
             (good.replace("total_sv 3", "total_sv 4"), "total_sv"),
             (good.replace("SV\n", ""), "SV")]
    for text, msg in cases:
        (tmp_path / "m.txt").write_text(text)
        with pytest.raises(pl.PlssvmError, match=msg):
            pl.plssvm_model_read(tmp_path / "m.txt")


def test_native_scaling_matches_oracle():
    rng = np.random.default_rng(9)
    X = rng.standard_normal((100, 12))
    X[:, 4] = 3.0  # constant feature -> lo
    fmin, fmax = pl.plssvm_scale_fit(X)
    rmin, rmax = ref.fit_scaling(X)
    assert np.array_equal(fmin, rmin) and np.array_equal(fmax, rmax)
    for lo, hi in [(-1.0, 1.0), (0.0, 1.0)]:
        assert np.array_equal(pl.plssvm_scale_apply(X, fmin, fmax, lo, hi), ref.apply_scaling(X, rmin, rmax, lo, hi))
    Z = rng.standard_normal((10, 12)) * 3  # outside the fitted range: no clamping
    assert np.array_equal(pl.plssvm_scale_apply(Z, fmin, fmax), ref.apply_scaling(Z, rmin, rmax))
    with pytest.raises(pl.PlssvmError):
        pl.plssvm_scale_apply(X, fmin, fmax, 1.0, 1.0)


# -------------------------------------------------------------------------------------- CLI
def _cli(*args, **kw):
    return subprocess.run([pl.cli_path(), *map(str, args)], capture_output=True, text=True, **kw)


def test_cli_scale_and_restore(tmp_path):
    rng = np.random.default_rng(4)
    X = rng.standard_normal((30, 5)) * 7
    y = np.where(rng.random(30) < 0.5, 1.0, -1.0)
    pl.plssvm_libsvm_write(tmp_path / "d.txt", X, y)
    r = _cli("scale", "-l", -1, "-u", 1, "-s", tmp_path / "range", tmp_path / "d.txt")
    assert r.returncode == 0, r.stderr
    Xs, ys, _ = ref.parse_libsvm(r.stdout)
    rmin, rmax = ref.fit_scaling(X)
    exp = ref.apply_scaling(X, rmin, rmax)
    assert np.array_equal(Xs, exp[:, :Xs.shape[1]]) and np.array_equal(ys, y)
    # restoring the saved ranges on the same file reproduces the output byte for byte
    r2 = _cli("scale", "-r", tmp_path / "range", tmp_path / "d.txt")
    assert r2.returncode == 0 and r2.stdout == r.stdout
    rng_lines = (tmp_path / "range").read_text().split("\n")
    assert rng_lines[0] == "x" and rng_lines[1] == "-1 1" and len([l for l in rng_lines[2:] if l]) == 5


def test_cli_usage_errors(tmp_path):
    assert _cli().returncode == 1
    assert _cli("train", "-t", 3, "x").returncode == 1  # sigmoid is rejected explicitly
    assert _cli("train").returncode == 1
    assert _cli("predict", "a", "b").returncode == 1
    r = _cli("train", tmp_path / "missing.txt")
    assert r.returncode == 2 and "missing.txt" in r.stderr
    (tmp_path / "one.txt").write_text("1 1:1\n1 1:2\n")
    assert _cli("train", tmp_path / "one.txt").returncode == 2  # one class only


def test_cli_links_dispatch():
    out = subprocess.run([os.path.join(os.path.dirname(pl.cli_path()), "plssvm-scale")], capture_output=True, text=True)
    assert out.returncode == 1 and "scale needs one data_file" in out.stderr
