"""Plain-Python oracle of the LIBSVM file formats and svm-scale -- TEST INFRASTRUCTURE ONLY
(same import rules as the rest of ``oracle/``: tests, smoke() and bench.py's reference legs).

Written from SPEC.md's io module and the paper's drop-in / dense-data statements
(P:52), one line at a time, no speed tricks:

* ``parse_libsvm``  -- S:109-117: "<label> <index>:<value> ...", 1-based strictly ascending
  indices, blank and '#' lines skipped, dense result with absent features 0, num_features = the
  largest index; labels returned RAW plus the distinct values in first-seen order.
* ``write_libsvm``  -- the same format, zero features omitted, reals as %.17g.
* ``write_model``   -- S:119-127: LIBSVM c_svc header, rho = -b (no "-0"), label / nr_sv, then
  "<alpha_i> <k>:<x_ik> ..." per point, the y = +1 points first, 17 significant digits.
* ``parse_model``   -- S:129-137.
* ``fit_scaling`` / ``apply_scaling`` -- S:139-147: min -> lo, max -> hi, constant -> lo, no clamping.

Parsing uses Python's float(), which rounds correctly, so a correct native parser agrees bit
for bit.
"""
from __future__ import annotations

import numpy as np


class FormatError(ValueError):
    pass


def _real(tok: str, line: int, what: str) -> float:
    try:
        v = float(tok)
    except ValueError:
        raise FormatError(f"line {line}: invalid {what} '{tok}'") from None
    if v != v or v in (float("inf"), float("-inf")):
        raise FormatError(f"line {line}: invalid {what} '{tok}'")
    return v


def parse_libsvm(text: str):
    """-> (X [m, d] float64, y_raw [m], distinct labels in first-seen order).  S:109-117."""
    labels, rows, distinct = [], [], []
    d = 0
    for ln, raw in enumerate(text.split("\n"), start=1):
        s = raw.strip(" \t\r\v\f")
        if s == "" or s.startswith("#"):
            continue
        toks = s.split()
        lab = _real(toks[0], ln, "label")
        if lab not in distinct:
            distinct.append(lab)
        feats = []
        prev = 0
        for t in toks[1:]:
            if ":" not in t:
                raise FormatError(f"line {ln}: invalid feature '{t}' (expected <index>:<value>)")
            si, sv = t.split(":", 1)
            try:
                k = int(si)
            except ValueError:
                raise FormatError(f"line {ln}: invalid feature '{t}' (expected <index>:<value>)") from None
            if k < 1:
                raise FormatError(f"line {ln}: feature index {k} < 1")
            if k <= prev:
                raise FormatError(f"line {ln}: indices must be ascending ({k} after {prev})")
            feats.append((k, _real(sv, ln, "value")))
            prev = k
        d = max(d, prev)
        labels.append(lab)
        rows.append(feats)
    if len(distinct) > 2:
        raise FormatError("more than two distinct labels")
    if not rows:
        raise FormatError("no data points")
    X = np.zeros((len(rows), d))
    for i, feats in enumerate(rows):
        for k, v in feats:
            X[i, k - 1] = v
    return X, np.array(labels, dtype=np.float64), distinct


def _num(v: float) -> str:
    v = float(v)
    if v == 0.0:
        v = 0.0  # no "-0"
    return "%.17g" % v


def _sparse(row) -> str:
    return "".join(f" {k + 1}:{_num(v)}" for k, v in enumerate(row) if v != 0.0)


def write_libsvm(X, y) -> str:
    return "".join(_num(y[i]) + _sparse(X[i]) + "\n" for i in range(len(y)))


_KERNEL_NAMES = {0: "linear", 1: "polynomial", 2: "rbf"}


def write_model(kernel, gamma, degree, coef0, X, alpha, b, y, labels) -> str:
    """S:119-127.  y in {+1, -1}; labels = (original label of +1, of -1)."""
    out = ["svm_type c_svc", f"kernel_type {_KERNEL_NAMES[kernel]}"]
    if kernel == 1:
        out.append(f"degree {int(degree)}")
    if kernel != 0:
        out.append(f"gamma {_num(gamma)}")
    if kernel == 1:
        out.append(f"coef0 {_num(coef0)}")
    npos = int(sum(1 for v in y if v == 1.0))
    out += ["nr_class 2", f"total_sv {len(y)}", f"rho {_num(-b)}", f"label {_num(labels[0])} {_num(labels[1])}",
            f"nr_sv {npos} {len(y) - npos}", "SV"]
    for cls in (1.0, -1.0):
        for i in range(len(y)):
            if y[i] == cls:
                out.append(_num(alpha[i]) + _sparse(X[i]))
    return "\n".join(out) + "\n"


def parse_model(text: str):
    """S:129-137 -> dict(kernel, gamma, degree, coef0, X, alpha, b, labels)."""
    lines = text.split("\n")
    hdr = {}
    i = 0
    while i < len(lines):
        s = lines[i].strip()
        i += 1
        if not s:
            continue
        if s == "SV":
            break
        key, _, rest = s.partition(" ")
        hdr[key] = rest.strip()
    else:
        raise FormatError("missing 'SV' line")
    for f in ("kernel_type", "nr_class", "total_sv", "rho", "label"):
        if f not in hdr:
            raise FormatError(f"missing field '{f}'")
    names = {v: k for k, v in _KERNEL_NAMES.items()}
    if hdr["kernel_type"] not in names:
        raise FormatError(f"unknown kernel_type '{hdr['kernel_type']}'")
    if int(float(hdr["nr_class"])) != 2:
        raise FormatError("nr_class must be 2")
    alpha, rows = [], []
    d = 0
    for ln in lines[i:]:
        s = ln.strip()
        if not s:
            continue
        toks = s.split()
        alpha.append(float(toks[0]))
        feats = [(int(t.split(":")[0]), float(t.split(":")[1])) for t in toks[1:]]
        d = max([d] + [k for k, _ in feats])
        rows.append(feats)
    X = np.zeros((len(rows), d))
    for r, feats in enumerate(rows):
        for k, v in feats:
            X[r, k - 1] = v
    kern = names[hdr["kernel_type"]]
    lab = [float(t) for t in hdr["label"].split()]
    rho = float(hdr["rho"])
    return dict(kernel=kern, gamma=float(hdr.get("gamma", 0.0)), degree=int(float(hdr.get("degree", 3))),
                coef0=float(hdr.get("coef0", 0.0)), X=X, alpha=np.array(alpha), b=-rho if rho != 0.0 else 0.0,
                labels=lab, total_sv=int(float(hdr["total_sv"])))


def fit_scaling(X):
    """per-feature (min, max) over all points."""
    return X.min(axis=0), X.max(axis=0)


def apply_scaling(X, fmin, fmax, lo=-1.0, hi=1.0):
    """x -> lo + (hi - lo) (x - min) / (max - min); constant features -> lo; no clamping."""
    out = np.empty_like(X, dtype=np.float64)
    for k in range(X.shape[1]):
        if fmax[k] == fmin[k]:
            out[:, k] = lo
        else:
            for i in range(X.shape[0]):
                out[i, k] = lo + (hi - lo) * (X[i, k] - fmin[k]) / (fmax[k] - fmin[k])
    return out
