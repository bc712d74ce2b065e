"""PRTS1 container bridge: read operators precomputed by
the reference onto the GPU, and export GPU-built operators in the
reference's on-disk format.

Format (reference `container.py:18-137, 156-235`, little-endian): an 80-byte
header {magic "PRTS1\\0\\0\\0", u32 version = 1, u32 flags, 32-byte mesh hash,
u32 sample count N, u32 K, u32 atlas parts m, u32 log2(grid side), 2 x u32
reserved}, then chunks {8-byte space-padded tag, u64 length, payload}:
BASIS (radial bases, f64), ATLAS (u32 part << 24 | cell per sample), one
TRANSFER per PCA term ({u32 k, f64 step1_keep, f64 step2_fraction}, then
{u32 n_cols, u64 nnz, f64 kept, f64 total, i64 step1 entries}, u32 cols,
i64 colptr, u32 rowidx, f32 vals), optional VIS / FOLD, and a JSON META.

This is host code (the container is file I/O, not the frame's hot path); the
operators it yields feed `DeviceTransfer.from_reference` (GPU layouts), and
`DeviceTransfer.to_reference` feeds `save_prts1`.
"""

from __future__ import annotations

import hashlib
import io
import json
import struct
from dataclasses import dataclass, field

import numpy as np

from .transfer import TransferOperator

MAGIC = b"PRTS1\x00\x00\x00"
VERSION = 1
HEADER = struct.Struct("<8sII32s6I")
CHUNK = struct.Struct("<8sQ")


class PRTS1Error(ValueError):
    pass


@dataclass
class RadialBasis:
    """The BASIS chunk: r nodes, (K, n_r) bases, singular values, eta, g,
    sigma box (the reference's DiffusionBasis fields)."""

    r_nodes: np.ndarray
    bases: np.ndarray
    singular_values: np.ndarray
    eta: float
    g: float
    sigma_box: tuple


@dataclass
class PRTS1:
    basis: RadialBasis
    part_of: np.ndarray       # (N,) u32
    cell_of: np.ndarray       # (N,) u32
    part_count: int
    grid_side: int
    operators: list           # [TransferOperator] * K
    step1_keep: float
    step2_fraction: float
    mesh_hash: bytes
    metadata: dict = field(default_factory=dict)
    chunks_skipped: tuple = ()

    @property
    def sample_count(self) -> int:
        return int(self.cell_of.size)

    def is_identity_geometry_image(self) -> bool:
        """Single-part atlas with cell i = sample i (the geometry images this
        repo renders)."""
        return (self.part_count == 1 and np.array_equal(self.part_of, np.zeros_like(self.part_of))
                and np.array_equal(self.cell_of, np.arange(self.cell_of.size, dtype=self.cell_of.dtype)))


def _tag(t: bytes) -> bytes:
    return t.ljust(8, b" ")


def _w(buf: io.BytesIO, a: np.ndarray, dtype: str):
    buf.write(np.ascontiguousarray(a, dtype).tobytes())


def _basis_bytes(b: RadialBasis) -> bytes:
    buf = io.BytesIO()
    r = np.asarray(b.r_nodes, np.float64)
    bases = np.asarray(b.bases, np.float64)
    sv = np.asarray(b.singular_values, np.float64)
    buf.write(struct.pack("<3I", r.size, bases.shape[0], sv.size))
    buf.write(struct.pack("<2d", float(b.eta), float(b.g)))
    buf.write(struct.pack("<4d", *[float(v) for v in b.sigma_box]))
    _w(buf, r, "<f8")
    _w(buf, bases, "<f8")
    _w(buf, sv, "<f8")
    return buf.getvalue()


def _operator_bytes(op: TransferOperator, k: int, keep: float, frac: float) -> bytes:
    buf = io.BytesIO()
    buf.write(struct.pack("<Idd", k, float(keep), float(frac)))
    cols = np.asarray(op.cols)
    rowidx = np.asarray(op.rowidx)
    buf.write(struct.pack("<IQ", cols.size, rowidx.size))
    buf.write(struct.pack("<ddq", float(op.kept_energy), float(op.total_energy),
                          int(op.step1_entries)))
    _w(buf, cols, "<u4")
    _w(buf, op.colptr, "<i8")
    _w(buf, rowidx, "<u4")
    _w(buf, op.vals, "<f4")
    return buf.getvalue()


def save_prts1(path, basis, operators, step1_keep: float, step2_fraction: float,
               side: int, mesh_hash: bytes = None, positions=None, metadata: dict = None,
               normals=None) -> None:
    """Write a PRTS1 container for a geometry image (identity single-part
    atlas of side x side cells). `basis` is any object with the BASIS fields
    (r_nodes, bases, singular_values, eta, g, sigma_box); `operators` are
    reference-format TransferOperators (e.g. DeviceTransfer.to_reference()).
    mesh_hash defaults to the reference's TriangleMesh.content_hash
    (surface.py:42-50) of the geometry image's grid mesh (vertices =
    positions, normals, grid triangles), so the reference's Scene accepts the
    container for that mesh."""
    n = side * side
    if mesh_hash is None:
        if positions is None or normals is None:
            raise PRTS1Error("need mesh_hash, or positions and normals of the geometry image")
        from .raster import TriangleMesh
        from .shadows import grid_triangles

        mesh_hash = TriangleMesh(np.asarray(positions, np.float64), np.asarray(normals, np.float64),
                                 grid_triangles(side)).content_hash()
    if len(mesh_hash) != 32:
        raise PRTS1Error("mesh hash must be 32 bytes (sha256)")
    level = int(np.log2(side)) if side > 1 else 0
    out = io.BytesIO()
    out.write(HEADER.pack(MAGIC, VERSION, 0, mesh_hash, n, len(operators), 1, level, 0, 0))

    def chunk(tag: bytes, payload: bytes):
        out.write(CHUNK.pack(_tag(tag), len(payload)))
        out.write(payload)

    rb = RadialBasis(basis.r_nodes, basis.bases, basis.singular_values, basis.eta, basis.g,
                     tuple(basis.sigma_box))
    chunk(b"BASIS", _basis_bytes(rb))
    records = np.arange(n, dtype=np.uint32)  # part 0 in the top byte, cell = sample
    chunk(b"ATLAS", struct.pack("<3I", 1, side, n) + records.astype("<u4").tobytes())
    for k, op in enumerate(operators):
        chunk(b"TRANSFER", _operator_bytes(op, k, step1_keep, step2_fraction))
    chunk(b"META", json.dumps(dict(metadata or {}), sort_keys=True).encode("utf-8"))
    with open(path, "wb") as fh:
        fh.write(out.getvalue())


def _read_operator(p: memoryview, off: int):
    n_cols, nnz = struct.unpack_from("<IQ", p, off)
    off += 12
    kept, total, s1 = struct.unpack_from("<ddq", p, off)
    off += 24

    def take(dtype, count):
        nonlocal off
        a = np.frombuffer(p, dtype, count, off)
        off += a.nbytes
        return a

    cols = take("<u4", n_cols).astype(np.uint32)
    colptr = take("<i8", n_cols + 1).astype(np.int64)
    rowidx = take("<u4", nnz).astype(np.uint32)
    vals = take("<f4", nnz).astype(np.float64)
    return TransferOperator(cols=cols, colptr=colptr, rowidx=rowidx, vals=vals,
                            kept_energy=float(kept), total_energy=float(total),
                            step1_entries=int(s1))


def load_prts1(path, expected_mesh_hash: bytes = None) -> PRTS1:
    """Parse a PRTS1 container (reference loader semantics: unknown chunks
    are an error; VIS / FOLD are recognised and skipped — the ambient folding
    path is outside this repo's scope)."""
    with open(path, "rb") as fh:
        data = memoryview(fh.read())
    if len(data) < HEADER.size:
        raise PRTS1Error(f"{path}: truncated header")
    magic, version, _flags, mesh_hash, n, k_count, m, level, _r0, _r1 = HEADER.unpack_from(data, 0)
    if magic != MAGIC:
        raise PRTS1Error(f"{path}: not a PRTS1 container")
    if version != VERSION:
        raise PRTS1Error(f"{path}: unsupported version {version}")
    if expected_mesh_hash is not None and mesh_hash != expected_mesh_hash:
        raise PRTS1Error(f"{path}: container was precomputed for a different mesh")
    basis = None
    atlas = None
    ops = {}
    keep = frac = None
    meta = {}
    skipped = []
    off = HEADER.size
    while off < len(data):
        if off + CHUNK.size > len(data):
            raise PRTS1Error(f"{path}: truncated chunk header")
        tag, length = CHUNK.unpack_from(data, off)
        off += CHUNK.size
        if off + length > len(data):
            raise PRTS1Error(f"{path}: truncated {tag.strip().decode()} chunk")
        p = data[off:off + length]
        off += length
        tag = bytes(tag).rstrip(b" ")
        if tag == b"BASIS":
            n_r, kk, n_sv = struct.unpack_from("<3I", p, 0)
            eta, g = struct.unpack_from("<2d", p, 12)
            box = struct.unpack_from("<4d", p, 28)
            o = 60
            r = np.frombuffer(p, "<f8", n_r, o).copy()
            o += 8 * n_r
            bases = np.frombuffer(p, "<f8", kk * n_r, o).reshape(kk, n_r).copy()
            o += 8 * kk * n_r
            sv = np.frombuffer(p, "<f8", n_sv, o).copy()
            basis = RadialBasis(r, bases, sv, float(eta), float(g), tuple(box))
        elif tag == b"ATLAS":
            parts, side, count = struct.unpack_from("<3I", p, 0)
            rec = np.frombuffer(p, "<u4", count, 12)
            atlas = (int(parts), int(side), (rec >> 24).astype(np.uint32),
                     (rec & 0xFFFFFF).astype(np.uint32))
        elif tag == b"TRANSFER":
            k, kp, fr = struct.unpack_from("<Idd", p, 0)
            ops[int(k)] = _read_operator(p, 20)
            keep, frac = float(kp), float(fr)
        elif tag in (b"VIS", b"FOLD"):
            skipped.append(tag.decode())
        elif tag == b"META":
            meta = json.loads(bytes(p).decode("utf-8"))
        else:
            raise PRTS1Error(f"{path}: unknown chunk {tag!r}")
    if basis is None or atlas is None or len(ops) != k_count:
        raise PRTS1Error(f"{path}: missing required chunks")
    parts, side, part_of, cell_of = atlas
    if cell_of.size != n or parts != m or (int(np.log2(side)) if side > 1 else 0) != level:
        raise PRTS1Error(f"{path}: header/chunk disagreement")
    return PRTS1(basis=basis, part_of=part_of, cell_of=cell_of, part_count=parts, grid_side=side,
                 operators=[ops[k] for k in range(k_count)], step1_keep=keep,
                 step2_fraction=frac, mesh_hash=bytes(mesh_hash), metadata=meta,
                 chunks_skipped=tuple(skipped))


def to_device(c: PRTS1, levels: int, device="cuda"):
    """Reference-built operators -> the GPU frame layout (DeviceTransfer).
    Requires the identity geometry-image atlas (what this repo renders)."""
    from .transfer import DeviceTransfer

    if not c.is_identity_geometry_image():
        raise PRTS1Error("only single-part identity atlases (geometry images) map to the GPU layout")
    return DeviceTransfer.from_reference(c.operators, c.grid_side, levels, device=device)


# ---------------------------------------------------------------------------
# GPU-native blocked layout, stored beside a container
# ---------------------------------------------------------------------------
# The reference's loader rejects unknown chunks (container.py:222-226), so the
# frame layout the transfer kernel streams (layout.KfrLayout: warp items,
# TMA batches of (column, term-mask) pair words + values) goes to a sidecar
# file <container>.kfr tied to the container's operators by a digest: loading
# it skips the layout build, and the container itself stays reference-valid.

KFR_MAGIC = "PRTSKFR1"
_KFR_ARRAYS = ("items", "lane_len", "lane_dst", "batch_off", "stream", "partial_row",
               "multi_info")


def operators_digest(operators) -> str:
    """sha256 over every operator's cols / colptr / rowidx / f32 vals."""
    h = hashlib.sha256()
    for op in operators:
        for a, dt in ((op.cols, "<u4"), (op.colptr, "<i8"), (op.rowidx, "<u4"), (op.vals, "<f4")):
            h.update(np.ascontiguousarray(a, dt).tobytes())
    return h.hexdigest()


def save_gpu_layout(path, layout, digest: str) -> None:
    """Write the kfr frame layout of an operator set (digest = operators_digest
    of the container's operators) as a sidecar .npz."""
    meta = {"magic": KFR_MAGIC, "K": layout.K, "n": layout.n, "n_items": layout.n_items,
            "n_partials": layout.n_partials, "stats": layout.stats, "digest": digest}
    arrays = {k: getattr(layout, k).cpu().numpy() for k in _KFR_ARRAYS}
    with open(path, "wb") as fh:
        np.savez(fh, meta=np.frombuffer(json.dumps(meta).encode("utf-8"), np.uint8), **arrays)


def load_gpu_layout(path, digest: str, device="cuda"):
    """Read a sidecar written by save_gpu_layout; PRTS1Error if it belongs to
    other operators (digest mismatch) or is not a kfr layout."""
    import torch

    from .layout import KFR_GROUP, KfrLayout

    with np.load(path) as z:
        meta = json.loads(bytes(z["meta"]).decode("utf-8"))
        if meta.get("magic") != KFR_MAGIC:
            raise PRTS1Error(f"{path}: not a kfr layout sidecar")
        if meta.get("digest") != digest:
            raise PRTS1Error(f"{path}: layout was built for different operators")
        t = {k: torch.as_tensor(z[k], device=device) for k in _KFR_ARRAYS}
    M = int(t["multi_info"].shape[0])
    dev = torch.device(device)
    return KfrLayout(
        K=meta["K"], n=meta["n"], n_items=meta["n_items"], n_partials=meta["n_partials"],
        items=t["items"], lane_len=t["lane_len"], lane_dst=t["lane_dst"],
        batch_off=t["batch_off"], stream=t["stream"],
        partials=torch.zeros((3 * KFR_GROUP, max(meta["n_partials"], 1)), dtype=torch.float64,
                             device=dev),
        partial_row=t["partial_row"], multi_info=t["multi_info"],
        multi_count=torch.zeros(M, dtype=torch.int32, device=dev),
        work=torch.zeros(2, dtype=torch.int32, device=dev), stats=meta["stats"])
