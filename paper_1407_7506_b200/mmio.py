"""MatrixMarket coordinate files -> SparseHermitian (host CSR, uploaded to the device CSR on
first use).  Same accepted formats, mirroring, duplicate summation and error behaviour as the
reference's ``read_matrix_market`` / ``write_matrix_market`` (problems.py:92-188):

* header ``%%MatrixMarket matrix coordinate {real|complex} {symmetric|hermitian}``; complex
  symmetric and non-coordinate / non-square inputs raise UnsupportedFormatError;
* 1-based indices, one stored triangle, entries mirrored (conjugated for Hermitian) and
  duplicates summed; malformed content raises ParseError(line, message) with the 1-based
  line number of the offending line;
* a non-real diagonal in a Hermitian file is a ParseError.

The entry lines are tokenised in bulk (numpy over the whole file: one C-level split and
float parse instead of a Python loop per entry); only files that fail the bulk checks are
re-scanned line by line to report the first offending line exactly as the reference does.
Values are parsed with Python's correctly rounded float conversion, so the matrix is
bit-identical to the reference's.
"""

from __future__ import annotations

import numpy as np

from .errors import ParseError, UnsupportedFormatError

__all__ = ["read_matrix_market", "write_matrix_market"]


def _parse_header(line):
    """problems.py:92-107."""
    parts = line.split()
    if len(parts) != 5 or parts[0] != "%%MatrixMarket":
        raise ParseError(1, "not a MatrixMarket header")
    _, obj, fmt, field, qualifier = (p.lower() for p in parts)
    if obj != "matrix" or fmt != "coordinate":
        raise UnsupportedFormatError(f"only coordinate matrices are supported, got {obj}/{fmt}")
    if field not in ("real", "complex"):
        raise UnsupportedFormatError(f"field {field!r} not supported (need real or complex)")
    if qualifier not in ("symmetric", "hermitian"):
        raise UnsupportedFormatError(f"qualifier {qualifier!r} not supported (need symmetric or hermitian)")
    if field == "complex" and qualifier == "symmetric":
        raise UnsupportedFormatError("complex symmetric files are not Hermitian")
    return field, qualifier


def _slow_scan(lines, field):
    """Line-by-line validation in the reference's order (problems.py:127-171); raises the
    first error with its line number, or returns the parsed entries."""
    size = None
    rows, cols, vals = [], [], []
    want = 4 if field == "complex" else 3
    lineno = 1
    for lineno, raw in enumerate(lines[1:], start=2):
        line = raw.strip()
        if not line or line.startswith("%"):
            continue
        parts = line.split()
        if size is None:
            if len(parts) != 3:
                raise ParseError(lineno, "size line must be 'rows cols nnz'")
            try:
                nr, nc, nnz = (int(p) for p in parts)
            except ValueError:
                raise ParseError(lineno, "size line must contain integers") from None
            if nr != nc:
                raise UnsupportedFormatError(f"matrix is {nr}x{nc}, need square")
            size = (nr, nnz)
            continue
        if len(parts) != want:
            raise ParseError(lineno, f"expected {want} fields, got {len(parts)}")
        try:
            i, j = int(parts[0]), int(parts[1])
            v = complex(float(parts[2]), float(parts[3])) if field == "complex" else float(parts[2])
        except ValueError:
            raise ParseError(lineno, "malformed entry") from None
        n = size[0]
        if not (1 <= i <= n and 1 <= j <= n):
            raise ParseError(lineno, f"index ({i}, {j}) out of range for n = {n}")
        if field == "complex" and i == j and v.imag != 0.0:
            raise ParseError(lineno, "hermitian matrix has a non-real diagonal entry")
        rows.append(i - 1)
        cols.append(j - 1)
        vals.append(v)
    if size is None:
        raise ParseError(lineno, "missing size line")
    if len(vals) != size[1]:
        raise ParseError(lineno, f"expected {size[1]} entries, found {len(vals)}")
    dt = np.complex128 if field == "complex" else np.float64
    return size[0], np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64), np.array(vals, dtype=dt)


def _fast_parse(lines, field):
    """Bulk tokenisation of the entry lines; None if anything needs the exact slow scan."""
    body = [ln for ln in lines[1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:
        return None
    head = body[0].split()
    if len(head) != 3:
        return None
    try:
        nr, nc, nnz = (int(p) for p in head)
    except ValueError:
        return None
    if nr != nc:
        return None
    want = 4 if field == "complex" else 3
    if len(body) - 1 != nnz:
        return None
    toks = " ".join(body[1:]).split()
    if len(toks) != want * nnz:
        return None
    try:
        arr = np.array(toks, dtype=object).reshape(nnz, want)
        rows = np.array(arr[:, 0], dtype=np.int64)
        cols = np.array(arr[:, 1], dtype=np.int64)
        re = np.asarray(arr[:, 2].astype(str), dtype=np.float64)
        im = np.asarray(arr[:, 3].astype(str), dtype=np.float64) if field == "complex" else None
    except (ValueError, TypeError):
        return None
    # a line with the right token count overall but a wrong count itself is caught here:
    if any(len(ln.split()) != want for ln in body[1:]):
        return None
    if rows.size and (rows.min() < 1 or cols.min() < 1 or rows.max() > nr or cols.max() > nr):
        return None
    if field == "complex":
        if np.any((rows == cols) & (im != 0.0)):
            return None
        vals = re + 1j * im
    else:
        vals = re
    return nr, rows - 1, cols - 1, vals


def read_matrix_market(path):
    """Read a MatrixMarket coordinate file into a SparseHermitian (problems.py:110-171)."""
    from .operators import SparseHermitian

    with open(path) as fh:
        lines = fh.readlines()
    if not lines:
        raise ParseError(1, "empty file")
    field, qualifier = _parse_header(lines[0])
    parsed = _fast_parse(lines, field)
    if parsed is None:
        parsed = _slow_scan(lines, field)
    n, rows, cols, vals = parsed
    return SparseHermitian.from_triangle(n, rows, cols, vals, qualifier)


def write_matrix_market(op, path):
    """Write the stored lower triangle in MatrixMarket coordinate format (problems.py:174-188),
    values in ``repr`` form (round-trip exact)."""
    field = "complex" if op.symmetry == "hermitian" else "real"
    rows, cols, vals = op.to_coo_lower()
    with open(path, "w") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate {field} {op.symmetry}\n")
        fh.write(f"{op.n} {op.n} {len(vals)}\n")
        if field == "complex":
            fh.writelines(f"{i + 1} {j + 1} {float(v.real)!r} {float(v.imag)!r}\n" for i, j, v in zip(rows, cols, vals))
        else:
            fh.writelines(f"{i + 1} {j + 1} {float(v)!r}\n" for i, j, v in zip(rows, cols, vals))
