"""Matrix Market coordinate I/O for the CSR path (drop-in for the reference's
read_matrix_market / write_matrix_market, sparse.py:292-428).

Accepted: ``%%MatrixMarket matrix coordinate <real|integer|complex|pattern>
<general|symmetric|hermitian|skew-symmetric>``.  Symmetric storage (lower
triangle) is expanded (mirror, conjugated for hermitian, negated for
skew-symmetric) and the result is assembled by ``CsrMatrix.from_coo``.
Every malformed input raises ``MatrixMarketError`` with the 1-based line
number the reference reports: header problems on line 1, size-line problems
on that line, entry problems on the entry's line, a count mismatch on the
last line, a duplicate on the line of its second occurrence (in sorted
order).  A ``pattern`` entry may carry an optional value (the reference's
pattern+values extension), else 1.0.
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from .errors import MatrixMarketError
from .sparse import CsrMatrix

FIELDS = ("real", "integer", "complex", "pattern")
SYMMETRIES = ("general", "symmetric", "hermitian", "skew-symmetric")


def _content(lines):
    """(1-based line number, stripped text) of every non-blank, non-comment line."""
    for no, raw in enumerate(lines, start=1):
        text = raw.strip()
        if text and not text.startswith("%"):
            yield no, text


def _header(first: str):
    tok = first.strip().split()
    if len(tok) != 5 or tok[0] != "%%MatrixMarket":
        raise MatrixMarketError("header must be '%%MatrixMarket matrix coordinate <field> <symmetry>'", line=1)
    obj, fmt, fld, sym = (t.lower() for t in tok[1:])
    if obj != "matrix" or fmt != "coordinate":
        raise MatrixMarketError(f"unsupported object/format {obj!r} {fmt!r}", line=1)
    if fld not in FIELDS:
        raise MatrixMarketError(f"unknown field {fld!r}", line=1)
    if sym not in SYMMETRIES:
        raise MatrixMarketError(f"unknown symmetry {sym!r}", line=1)
    return fld, sym


def _value(fld: str, parts, no: int, text: str):
    try:
        if fld == "complex":
            if len(parts) != 4:
                raise MatrixMarketError("complex entry needs 're im'", line=no)
            return complex(float(parts[2]), float(parts[3]))
        if fld == "pattern":
            return float(parts[2]) if len(parts) >= 3 else 1.0
        if len(parts) != 3:
            raise MatrixMarketError("entry needs exactly one value", line=no)
        return float(parts[2])
    except ValueError:
        raise MatrixMarketError(f"bad numeric value in {text!r}", line=no) from None


def read_matrix_market(path) -> CsrMatrix:
    with open(path) as fh:
        lines = fh.readlines()
    if not lines:
        raise MatrixMarketError("empty file", line=1)
    fld, sym = _header(lines[0])
    body = _content(lines[1:])

    size = None
    for no, text in body:
        no += 1  # _content counted from the second line
        parts = text.split()
        if len(parts) != 3:
            raise MatrixMarketError("size line must be 'nrows ncols nnz'", line=no)
        try:
            size = tuple(int(p) for p in parts)
        except ValueError:
            raise MatrixMarketError("size line must be integer", line=no) from None
        size_line = no
        break
    if size is None:
        raise MatrixMarketError("missing size line", line=len(lines))
    nrows, ncols, declared = size
    if min(size) < 0:
        raise MatrixMarketError("negative dimension", line=size_line)
    if sym != "general" and nrows != ncols:
        raise MatrixMarketError(f"{sym} matrix must be square", line=size_line)

    rows, cols, vals, where = [], [], [], []
    for no, text in body:
        no += 1
        if len(rows) == declared:
            raise MatrixMarketError(f"more than the declared {declared} entries", line=no)
        parts = text.split()
        try:
            i, j = int(parts[0]) - 1, int(parts[1]) - 1
        except (ValueError, IndexError):
            raise MatrixMarketError("entry must start with two integer indices", line=no) from None
        if not (0 <= i < nrows and 0 <= j < ncols):
            raise MatrixMarketError(f"index ({i + 1},{j + 1}) out of bounds", line=no)
        v = _value(fld, parts, no, text)
        if sym != "general" and i < j:
            raise MatrixMarketError(
                f"{sym} storage requires lower-triangle entries (got row {i + 1} < col {j + 1})", line=no)
        if sym == "hermitian" and i == j and fld == "complex" and v.imag != 0.0:
            raise MatrixMarketError("hermitian diagonal must be real", line=no)
        rows.append(i)
        cols.append(j)
        vals.append(v)
        where.append(no)
    if len(rows) != declared:
        raise MatrixMarketError(f"declared {declared} entries but found {len(rows)}", line=len(lines))

    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    v = np.asarray(vals, dtype=np.complex128 if fld == "complex" else np.float64)
    if len(r) > 1:
        order = np.lexsort((c, r))
        same = (np.diff(r[order]) == 0) & (np.diff(c[order]) == 0)
        if same.any():
            k = int(np.flatnonzero(same)[0]) + 1
            raise MatrixMarketError(f"duplicate entry ({r[order[k]] + 1},{c[order[k]] + 1})",
                                    line=where[int(order[k])])
    if sym != "general":
        off = r != c
        mirror = v[off]
        if sym == "hermitian":
            mirror = np.conj(mirror)
        elif sym == "skew-symmetric":
            mirror = -mirror
        r, c = np.concatenate([r, c[off]]), np.concatenate([c, r[off]])
        v = np.concatenate([v, mirror])
    return CsrMatrix.from_coo(nrows, ncols, r, c, v)


def write_matrix_market(a: CsrMatrix, path, comment: Optional[str] = None) -> None:
    """Coordinate 'general' storage, values with 17 significant digits."""
    cplx = np.iscomplexobj(a.vals)
    rows = np.repeat(np.arange(a.nrows), np.diff(a.row_ptr)) + 1
    cols = np.asarray(a.col_idx, dtype=np.int64) + 1
    out = [f"%%MatrixMarket matrix coordinate {'complex' if cplx else 'real'} general\n"]
    if comment:
        out.append(f"% {comment}\n")
    out.append(f"{a.nrows} {a.ncols} {a.nnz}\n")
    if cplx:
        out.extend(f"{i} {j} {z.real:.17g} {z.imag:.17g}\n" for i, j, z in zip(rows, cols, a.vals))
    else:
        out.extend(f"{i} {j} {x:.17g}\n" for i, j, x in zip(rows, cols, a.vals))
    with open(path, "w") as fh:
        fh.writelines(out)
