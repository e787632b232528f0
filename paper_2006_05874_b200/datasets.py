"""Datasets feeding the solvers (proj/include/ihs/datasets.hpp): CSV and
libsvm/svmlight loaders with the reference's validation order and error types,
and the seeded synthetic spectra generator.

generate_synthetic draws its Gaussian factors from the reference's RNG streams
(make_stream(seed, 10 / 11 / 12 / 13), fill_gaussian — generated on the device,
bit-identical to std::mt19937_64 + libstdc++'s normal_distribution) and takes
the orthonormal factors from a Householder QR (numpy/LAPACK in place of Eigen's
HouseholderQR: the same reflector convention, equal to it up to rounding).
The singular values are exactly the requested spectrum either way.
"""
from __future__ import annotations

import enum
import math
import re
from dataclasses import dataclass

import numpy as np

from . import ihs


class DatasetSource(enum.IntEnum):  # datasets.hpp:19
    CSVFile = 0
    LibsvmFile = 1
    SyntheticExp = 2
    SyntheticPoly = 3


class SyntheticKind(enum.IntEnum):  # datasets.hpp:20
    Exp = 0
    Poly = 1


@dataclass
class Dataset:  # datasets.hpp:22-30
    A: np.ndarray
    b: np.ndarray
    source: DatasetSource = DatasetSource.CSVFile
    provenance: str = ""

    def n(self) -> int:
        return self.A.shape[0]

    def d(self) -> int:
        return self.A.shape[1]


def _stream_normals(seed: int, tag: int, count: int, stddev: float) -> np.ndarray:
    # fill_gaussian(v, make_stream(seed, tag), stddev) for a vector / column-major matrix (rng.hpp:35-40)
    return ihs.fill_gaussian(ihs.derive_seed(seed, tag), count, 1, stddev).reshape(-1, order="F")


def orthonormal_factor(rows: int, cols: int, seed: int, tag: int) -> np.ndarray:
    """datasets.hpp:32-38: orthonormal columns from the thin QR of a seeded Gaussian matrix."""
    G = ihs.fill_gaussian(ihs.derive_seed(seed, tag), rows, cols, 1.0)
    Q, _ = np.linalg.qr(G, mode="reduced")
    return Q


def synthetic_spectrum(kind: SyntheticKind, d: int) -> np.ndarray:
    """datasets.hpp:52-58: 0.95^j (Exp) or 1/j (Poly), j = 1..d."""
    j = np.arange(1, d + 1, dtype=np.float64)
    return np.power(0.95, j) if kind == SyntheticKind.Exp else 1.0 / j


def matrix_with_spectrum(n: int, d: int, sigma: np.ndarray, seed: int) -> np.ndarray:
    """datasets.hpp:40-50: A = U diag(sigma) V^T with seeded orthonormal factors."""
    if n < d or d < 1:
        raise ihs.InvalidInput("matrix_with_spectrum: need n >= d >= 1")
    if sigma.size != d:
        raise ihs.InvalidInput("matrix_with_spectrum: spectrum length must equal d")
    U = orthonormal_factor(n, d, seed, 10)
    V = orthonormal_factor(d, d, seed, 11)
    return np.asfortranarray((U * sigma) @ V.T)


def generate_synthetic(kind: SyntheticKind, n: int, d: int, seed: int) -> Dataset:
    """datasets.hpp:63-80: planted model b = A x_pl + noise, x_pl ~ N(0, 1/d), noise ~ N(0, 1/n)."""
    if n < d or d < 1:
        raise ihs.InvalidInput("generate_synthetic: need n >= d >= 1")
    A = matrix_with_spectrum(n, d, synthetic_spectrum(kind, d), seed)
    x_pl = _stream_normals(seed, 12, d, 1.0 / math.sqrt(d))
    noise = _stream_normals(seed, 13, n, 1.0 / math.sqrt(n))
    b = A @ x_pl + noise
    name = "exp" if kind == SyntheticKind.Exp else "poly"
    return Dataset(A, b, DatasetSource.SyntheticExp if kind == SyntheticKind.Exp else DatasetSource.SyntheticPoly,
                   f"synthetic-{name} n={n} d={d} seed={seed}")


# ------------------------------------------------------------------ text loaders
def _parse_number(tok: str, line: int) -> float:
    """datasets.hpp:84-96: std::stod semantics — leading whitespace and a numeric prefix, then only
    trailing whitespace."""
    s = tok.lstrip()
    m = re.match(r"[+-]?((\d+\.?\d*|\.\d+)([eE][+-]?\d+)?|inf(inity)?|nan(\([^)]*\))?|0[xX][0-9a-fA-F.]+([pP][+-]?\d+)?)",
                 s, re.IGNORECASE)
    if not m:
        raise ihs.ParseError(f"malformed number '{tok}'", line)
    rest = s[m.end():]
    if rest.strip():
        raise ihs.ParseError(f"trailing characters in number '{tok}'", line)
    txt = m.group(0)
    try:
        return float.fromhex(txt) if txt.lower().lstrip("+-").startswith("0x") else float(txt)
    except ValueError:
        raise ihs.ParseError(f"malformed number '{tok}'", line) from None


def _lines(path: str, who: str):
    try:
        with open(path, "r") as f:
            return f.read().split("\n")
    except OSError:
        raise ihs.InvalidInput(f"{who}: cannot open '{path}'") from None


def load_csv(path: str) -> Dataset:
    """datasets.hpp:106-141: one observation per row, last column = b."""
    lines = _lines(path, "load_csv")
    if lines and lines[-1] == "":
        lines.pop()  # std::getline yields no final empty line after a trailing newline
    rows = []
    lineno = 0
    for line in lines:
        lineno += 1
        if not line.strip():
            continue
        toks = line.split(",")
        if line.endswith(","):
            toks.pop()  # std::getline(ss, tok, ',') does not produce a trailing empty token
        row = [_parse_number(tok, lineno) for tok in toks]
        if len(row) < 2:
            raise ihs.ParseError("need at least one feature column and one label", lineno)
        if rows and len(row) != len(rows[0]):
            raise ihs.ShapeError(f"load_csv: row {lineno} has {len(row)} columns, expected {len(rows[0])}")
        rows.append(row)
    if not rows:
        raise ihs.ParseError(f"load_csv: no data rows in '{path}'", lineno)
    M = np.asarray(rows, dtype=np.float64)
    A, b = np.asfortranarray(M[:, :-1]), np.ascontiguousarray(M[:, -1])
    if not (np.all(np.isfinite(A)) and np.all(np.isfinite(b))):
        raise ihs.InvalidInput("load_csv: non-finite entries")
    return Dataset(A, b, DatasetSource.CSVFile, "csv:" + path)


def load_libsvm(path: str) -> Dataset:
    """datasets.hpp:145-193: 'label index:value ...', 1-based indices, densified with zeros."""
    lines = _lines(path, "load_libsvm")
    if lines and lines[-1] == "":
        lines.pop()
    labels, feats = [], []
    d = 0
    lineno = 0
    for line in lines:
        lineno += 1
        if not line.strip():
            continue
        toks = line.split()
        if not toks:
            raise ihs.ParseError("missing label", lineno)
        labels.append(_parse_number(toks[0], lineno))
        row = {}
        for tok in toks[1:]:
            colon = tok.find(":")
            if colon <= 0 or colon + 1 == len(tok):
                raise ihs.ParseError(f"expected 'index:value', got '{tok}'", lineno)
            head = tok[:colon]
            mi = re.match(r"\s*[+-]?\d+", head)
            if not mi:
                raise ihs.ParseError(f"malformed feature index in '{tok}'", lineno)
            idx = int(mi.group(0))  # std::stol: the numeric prefix
            if idx < 1:
                raise ihs.ParseError(f"feature indices are 1-based, got {idx}", lineno)
            row[idx - 1] = _parse_number(tok[colon + 1:], lineno)
            d = max(d, idx)
        feats.append(row)
    if not labels:
        raise ihs.ParseError(f"load_libsvm: no data rows in '{path}'", lineno)
    if d == 0:
        raise ihs.ParseError("load_libsvm: no features present", lineno)
    A = np.zeros((len(labels), d), order="F")
    for i, row in enumerate(feats):
        for j, v in row.items():
            A[i, j] = v
    b = np.asarray(labels, dtype=np.float64)
    if not (np.all(np.isfinite(A)) and np.all(np.isfinite(b))):
        raise ihs.InvalidInput("load_libsvm: non-finite entries")
    return Dataset(A, b, DatasetSource.LibsvmFile, "libsvm:" + path)
