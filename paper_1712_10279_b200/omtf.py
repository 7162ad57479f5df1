"""File formats the CLI needs: OMTF density / flux files
(S/fields.py:297-365), CSV scalar fields, channel-graph JSON (S/graph.py:137-156)
and matrix-set JSON (S/lindblad.py:189-215).  Byte layout identical to the
reference: magic ``OMTF1``, three little-endian uint32 (kind, n, k), then
row-major float64 payload, complex entries interleaved (re, im)."""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from .errors import ValidationError
from .fields import MatrixDensity, ScalarDensity, VectorDensity
from .graph import TransportGraph
from .lindblad import LindbladSet

MAGIC = b"OMTF1"
KIND_SCALAR, KIND_VECTOR, KIND_MATRIX_REAL, KIND_MATRIX_COMPLEX = 0, 1, 2, 3
GRAPH_FORMAT_VERSION = 1
LINDBLAD_FORMAT_VERSION = 1


def _payload(kind, arr):
    if kind == KIND_MATRIX_COMPLEX:
        arr = np.stack([arr.real, arr.imag], axis=-1)
    elif kind == KIND_MATRIX_REAL:
        arr = np.real(arr)
    return np.ascontiguousarray(arr, dtype="<f8").tobytes()


def _write(path, kind, n, k, arr):
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<III", kind, n, k))
        fh.write(_payload(kind, arr))


def write_omtf(path, field) -> None:
    """Density field -> OMTF file (S/fields.py:297-319)."""
    if isinstance(field, ScalarDensity):
        _write(path, KIND_SCALAR, field.n, 1, field.values)
    elif isinstance(field, VectorDensity):
        _write(path, KIND_VECTOR, field.n, field.k, field.values)
    elif isinstance(field, MatrixDensity):
        kind = KIND_MATRIX_REAL if np.all(field.values.imag == 0) else KIND_MATRIX_COMPLEX
        _write(path, kind, field.n, field.k, field.values)
    else:
        raise ValidationError(f"cannot write object of type {type(field).__name__}")


def write_flux(prefix, ux, uy, kind_hint: str) -> None:
    """Signed flux components as raw OMTF-framed arrays, one file per axis
    (``<prefix>.ux.omtf`` / ``.uy.omtf``), as the reference CLI dumps them."""
    base = Path(prefix)
    for suffix, arr in ((".ux.omtf", ux), (".uy.omtf", uy)):
        arr = np.asarray(arr)
        if kind_hint == "scalar":
            kind, k = KIND_SCALAR, 1
        elif kind_hint == "vector":
            kind, k = KIND_VECTOR, arr.shape[-1]
        else:
            k = arr.shape[-1]
            kind = KIND_MATRIX_REAL if np.all(arr.imag == 0) else KIND_MATRIX_COMPLEX
        target = base.with_suffix(base.suffix + suffix) if base.suffix else \
            base.parent / (base.name + suffix)
        _write(target, kind, arr.shape[0], k, arr)


def read_omtf(path):
    """OMTF file -> density of the matching kind (S/fields.py:322-349)."""
    raw = Path(path).read_bytes()
    if len(raw) < len(MAGIC) + 12 or raw[: len(MAGIC)] != MAGIC:
        raise ValidationError(f"{path}: not an OMTF file")
    kind, n, k = struct.unpack_from("<III", raw, len(MAGIC))
    body = np.frombuffer(raw, dtype="<f8", offset=len(MAGIC) + 12)
    shapes = {KIND_SCALAR: (n, n), KIND_VECTOR: (n, n, k), KIND_MATRIX_REAL: (n, n, k, k),
              KIND_MATRIX_COMPLEX: (n, n, k, k, 2)}
    if kind not in shapes:
        raise ValidationError(f"{path}: unknown OMTF kind {kind}")
    shape = shapes[kind]
    if body.size != int(np.prod(shape)):
        raise ValidationError(f"{path}: payload size {body.size} != expected {int(np.prod(shape))}")
    body = body.reshape(shape)
    if kind == KIND_SCALAR:
        return ScalarDensity(body)
    if kind == KIND_VECTOR:
        return VectorDensity(body)
    if kind == KIND_MATRIX_REAL:
        return MatrixDensity(body.astype(np.complex128))
    return MatrixDensity(body[..., 0] + 1j * body[..., 1])


def read_density(path):
    """OMTF, or CSV (n rows of n values) for scalar fields."""
    path = Path(path)
    if path.suffix.lower() == ".csv":
        arr = np.loadtxt(path, delimiter=",", ndmin=2)
        if arr.shape[0] != arr.shape[1]:
            raise ValidationError(f"{path}: CSV must be square, got {arr.shape}")
        return ScalarDensity(arr)
    return read_omtf(path)


def load_graph(path) -> TransportGraph:
    """{k, edges (1-indexed pairs), costs} JSON."""
    data = json.loads(Path(path).read_text())
    try:
        edges = [(int(a) - 1, int(b) - 1) for a, b in data["edges"]]
        return TransportGraph(int(data["k"]), edges, data["costs"])
    except (KeyError, TypeError, ValueError) as exc:
        raise ValidationError(f"{path}: malformed graph file ({exc})") from exc


def save_graph(path, g: TransportGraph) -> None:
    Path(path).write_text(json.dumps({
        "format_version": GRAPH_FORMAT_VERSION, "k": g.k,
        "edges": [[a + 1, b + 1] for a, b in g.edges],
        "costs": [float(c) for c in g.costs]}, indent=2) + "\n")


def load_lindblad(path) -> LindbladSet:
    """{k, ell, matrices: per matrix a row-major list of [re, im]} JSON."""
    data = json.loads(Path(path).read_text())
    try:
        k, ell = int(data["k"]), int(data["ell"])
        mats = np.empty((ell, k, k), dtype=np.complex128)
        for s, flat in enumerate(data["matrices"]):
            if len(flat) != k * k:
                raise ValueError(f"matrix {s} has {len(flat)} entries, expected {k * k}")
            mats[s] = np.array([complex(re, im) for re, im in flat]).reshape(k, k)
    except (KeyError, TypeError, ValueError) as exc:
        raise ValidationError(f"{path}: malformed matrix-set file ({exc})") from exc
    return LindbladSet(mats)


def save_lindblad(path, L: LindbladSet) -> None:
    Path(path).write_text(json.dumps({
        "format_version": LINDBLAD_FORMAT_VERSION, "k": L.k, "ell": L.ell,
        "matrices": [[[float(z.real), float(z.imag)] for z in m.ravel()] for m in L.matrices]},
        indent=2) + "\n")
