"""Build frame layout v6 (csrc/stream6.cu) from the canonical tile-major CSR
operator, on the GPU: per-SM units of consecutive tiles, items = (unit,
column band[, split]) with entries sorted by (row, k, column) and packed as
{u32 (row_local << 4 | k) << 11 | band-local column, f32 value}.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

SLOTS = 3
SLOT_BYTES = 24576
BAND_WIDTH = 1024  # <= 2048 (11 column bits)
COL_BITS = 11
ITEM_DTYPE = np.dtype([("off", "<u8"), ("n", "<u4"), ("band", "<u2"), ("pad", "<u2")])


@dataclass
class V6Layout:
    slot_bytes: int
    band_width: int
    units: int
    unit_tile0: torch.Tensor
    unit_ntiles: torch.Tensor
    unit_item0: torch.Tensor
    unit_nitems: torch.Tensor
    items: torch.Tensor
    stream: torch.Tensor
    n_items: int
    stream_bytes: int
    max_unit_items: int
    max_unit_rows: int


def build_v6(dt, slot_bytes: int = SLOT_BYTES, band_width: int = BAND_WIDTH,
             n_sm: int = None) -> V6Layout:
    dev = dt.rowptr.device
    if n_sm is None:
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    n, K = dt.n, dt.K
    if K > 16:
        raise ValueError("v6 packs k in 4 bits (K <= 16)")
    BW = min(band_width, n)
    if BW > (1 << COL_BITS):
        raise ValueError("band_width exceeds the 11 column bits")
    NB = (n + BW - 1) // BW
    T2 = (1 << dt.levels) ** 2
    ntiles = n // T2
    G = -(-ntiles // n_sm)
    R_unit = G * T2
    if R_unit > 512:
        raise ValueError("more than 512 rows per unit (9 row bits)")
    units = -(-ntiles // G)
    cap = slot_bytes // 8
    cap -= cap & 1
    rp = dt.rowptr.cpu().numpy()
    row_len = rp[:, 1:] - rp[:, :-1]
    nnz = dt.nnz
    k_of = torch.repeat_interleave(torch.arange(K, device=dev),
                                   torch.as_tensor(row_len.sum(axis=1), device=dev))
    row_of = torch.repeat_interleave(
        torch.arange(n, device=dev).repeat(K), torch.as_tensor(row_len.reshape(-1), device=dev))
    col = dt.cols.to(torch.int64) & 0xFFFFFFFF
    band = col // BW
    col_local = col % BW
    unit = row_of // R_unit
    row_local = row_of % R_unit
    meta = (((row_local << 4) | k_of) << COL_BITS) | col_local
    # stream order: (unit, band, row_local, k, col)
    key = ((unit * NB + band) << 32) | meta
    order = torch.argsort(key)
    ub = (unit * NB + band)[order]
    idx = torch.arange(nnz, device=dev)
    grp_flag = torch.ones(nnz, dtype=torch.bool, device=dev)
    grp_flag[1:] = ub[1:] != ub[:-1]
    grp_first = torch.cummax(torch.where(grp_flag, idx, torch.zeros_like(idx)), 0).values
    gpos = idx - grp_first
    sub = gpos // cap
    item_key = ub * 65536 + sub
    ik_flag = torch.ones(nnz, dtype=torch.bool, device=dev)
    ik_flag[1:] = item_key[1:] != item_key[:-1]
    item_id = torch.cumsum(ik_flag.to(torch.int64), 0) - 1
    n_items = int(item_id[-1].item()) + 1 if nnz else 0
    item_n = torch.bincount(item_id, minlength=n_items).cpu().numpy().astype(np.int64)
    first_e = torch.nonzero(ik_flag).squeeze(1)
    item_ub = ub[first_e].cpu().numpy()
    item_unit = item_ub // NB
    item_band = item_ub % NB
    item_bytes = 8 * (item_n + (item_n & 1))
    item_off = np.zeros(n_items + 1, np.int64)
    np.cumsum(item_bytes, out=item_off[1:])
    total = int(item_off[-1])
    stream = torch.zeros(max(total, 16), dtype=torch.uint8, device=dev)
    off_d = torch.as_tensor(item_off[:-1], device=dev)
    dst = off_d[item_id] // 8 + (gpos - sub * cap)
    vbits = dt.vals.view(torch.int32).to(torch.int64)[order] & 0xFFFFFFFF
    stream.view(torch.int64)[dst] = meta[order] | (vbits << 32)
    unit_nitems = np.bincount(item_unit, minlength=units)
    unit_item0 = np.zeros(units, np.int64)
    unit_item0[1:] = np.cumsum(unit_nitems)[:-1]
    items = np.zeros(n_items, ITEM_DTYPE)
    items["off"] = item_off[:-1]
    items["n"] = item_n
    items["band"] = item_band
    unit_tile0 = np.arange(units) * G
    unit_ntiles = np.minimum(G, ntiles - unit_tile0)
    return V6Layout(
        slot_bytes=slot_bytes, band_width=BW, units=units,
        unit_tile0=torch.as_tensor(unit_tile0.astype(np.int32), device=dev),
        unit_ntiles=torch.as_tensor(unit_ntiles.astype(np.int32), device=dev),
        unit_item0=torch.as_tensor(unit_item0.astype(np.int32), device=dev),
        unit_nitems=torch.as_tensor(unit_nitems.astype(np.int32), device=dev),
        items=torch.as_tensor(items.view(np.uint8), device=dev), stream=stream,
        n_items=n_items, stream_bytes=total,
        max_unit_items=int(unit_nitems.max()) if units else 0, max_unit_rows=R_unit)


def launch_v6(lay: V6Layout, dt, x, g, positions, normals, cam, material, vk, scatter, radiance,
              radiance_unclamped, stream=None):
    _lib.call("sss_transfer_v6", dt.K, dt.side, dt.levels, lay.band_width, lay.slot_bytes,
              lay.units, lay.max_unit_items, lay.max_unit_rows, _lib.ptr(lay.unit_tile0),
              _lib.ptr(lay.unit_ntiles), _lib.ptr(lay.unit_item0), _lib.ptr(lay.unit_nitems),
              _lib.ptr(lay.items), _lib.ptr(lay.stream), _lib.ptr(x), _lib.ptr(g),
              _lib.ptr(positions), _lib.ptr(normals), _lib.ptr(cam), _lib.ptr(material),
              _lib.ptr(vk), _lib.ptr(scatter), _lib.ptr(radiance), _lib.ptr(radiance_unclamped),
              _lib.stream_ptr(stream))
