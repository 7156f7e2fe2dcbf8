"""BAL text I/O: ``parse_bal`` / ``serialize_bal`` (dba/bal_io.hpp:78-209).

Both run in libdbag.so (csrc/bal.hpp): the text is scanned in memory with the
reference's token rules, validation, messages and line numbers; reals are
parsed in double and cast to the problem's Scalar exactly as
``parse_bal<Scalar>`` casts them; emission prints every real with "%.16e".
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Union

import numpy as np

from . import _native as N
from .dba import BAProblem, _check

PathOrText = Union[str, bytes, os.PathLike]


def _read(source: PathOrText) -> bytes:
    if isinstance(source, bytes):
        return source
    with open(source, "rb") as f:
        return f.read()


def parse_bal(source: PathOrText, dtype=np.float64, warnings: Optional[List[str]] = None) -> BAProblem:
    """Parses BAL text (a path, or the bytes themselves) into a BAProblem of
    ``dtype``. Raises ParseError("line L: ...") with ``.line`` on malformed
    input; problem.validate() warnings (unreferenced nodes, non-positive
    focal) are appended to ``warnings`` when given (dba/bal_io.hpp:139-142)."""
    text = _read(source)
    lib = N.lib()
    h = C.c_void_p()
    _check(lib.dbag_bal_parse(text, len(text), C.byref(h)))
    try:
        m, n, nobs = C.c_int32(), C.c_int32(), C.c_int64()
        _check(lib.dbag_bal_counts(h, C.byref(m), C.byref(n), C.byref(nobs)))
        cams = np.empty((m.value, 9))
        pts = np.empty((n.value, 3))
        cid = np.empty(nobs.value, np.int32)
        pid = np.empty(nobs.value, np.int32)
        px = np.empty(nobs.value)
        py = np.empty(nobs.value)
        _check(lib.dbag_bal_copy(h, cams.ctypes.data, pts.ctypes.data, cid.ctypes.data, pid.ctypes.data,
                                 px.ctypes.data, py.ctypes.data))
    finally:
        lib.dbag_bal_free(h)
    problem = BAProblem.from_arrays(cams, pts, cid, pid, np.stack([px, py], axis=1), dtype=dtype)
    if warnings is not None:
        warnings.extend(problem.validate())
    return problem


def format_bal(problem: BAProblem) -> bytes:
    """The BAL text serialize_bal writes for ``problem``."""
    lib = N.lib()
    s = problem.c_struct()
    buf, n = C.c_void_p(), C.c_int64()
    _check(lib.dbag_bal_format(problem.precision, C.byref(s), C.byref(buf), C.byref(n)))
    try:
        return C.string_at(buf.value, n.value)
    finally:
        lib.dbag_free_text(buf)


def serialize_bal(problem: BAProblem, out=None) -> Optional[bytes]:
    """serialize_bal (dba/bal_io.hpp:158-209): writes to ``out`` (a path or a
    binary/text stream); returns the bytes when ``out`` is None."""
    text = format_bal(problem)
    if out is None:
        return text
    if isinstance(out, (str, os.PathLike)):
        with open(out, "wb") as f:
            f.write(text)
    elif hasattr(out, "buffer"):
        out.buffer.write(text)
    else:
        try:
            out.write(text)
        except TypeError:
            out.write(text.decode())
    return None
