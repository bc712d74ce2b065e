"""Build frame layout v5 (csrc/stream4.cu) from the canonical tile-major CSR
operator, on the GPU: per-SM units, virtual threads, self-describing items
(one per unit x column band [x split]) carrying every PCA term.

Stream order inside an item: virtual thread, then k, then column. A row's
(band, k) segment is cut into its m_r virtual threads' pieces with
piece(p) = ((p + 1) m - 1) // len. The order is produced by one device sort
on a composite key; headers (per-thread counts + warp bases) are small
bincounts.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

NW = 16  # consumer warps (csrc/stream4.cu: kV4Warps)
TPU = NW * 32
SLOTS = 4
HDR = (2 * (NW + 1) + 2 * TPU + 15) & ~15  # u16 warp bases + u16 counts, 16-B padded
MAXCNT = 65535
SLOT_BYTES = 32768
BAND_WIDTH = 1024  # w0 ids per x band (3 x 1024 doubles per buffer, double-buffered)

ITEM_DTYPE = np.dtype([("off", "<u8"), ("bytes", "<u4"), ("band", "<u2"), ("pad", "<u2")])


@dataclass
class V4Layout:
    slot_bytes: int
    band_width: int
    units: int
    unit_tile0: torch.Tensor
    unit_ntiles: torch.Tensor
    unit_item0: torch.Tensor
    unit_nitems: torch.Tensor
    items: torch.Tensor  # uint8 view of ITEM_DTYPE records
    stream: torch.Tensor  # uint8, 16-B aligned
    vrow_first: torch.Tensor  # int16 (u16) per unit R+1
    n_items: int
    stream_bytes: int
    header_bytes: int
    max_unit_items: int


def _threads_per_row(row_tot: np.ndarray, R: int) -> np.ndarray:
    """1 thread per row + the spare ones proportional to row length."""
    m = np.ones(R, np.int64)
    spare = TPU - R
    tot = float(row_tot.sum())
    if spare > 0 and tot > 0:
        share = spare * row_tot / tot
        extra = np.floor(share).astype(np.int64)
        rem = spare - int(extra.sum())
        if rem > 0:
            extra[np.argsort(-(share - extra), kind="stable")[:rem]] += 1
        m += extra
    return m


def build_v4(dt, slot_bytes: int = SLOT_BYTES, band_width: int = BAND_WIDTH,
             n_sm: int = None) -> V4Layout:
    dev = dt.rowptr.device
    if n_sm is None:
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    n, K = dt.n, dt.K
    BW = min(band_width, n)
    NB = (n + BW - 1) // BW
    T2 = (1 << dt.levels) ** 2
    ntiles = n // T2
    G = -(-ntiles // n_sm)
    if G * T2 > TPU:
        raise ValueError(f"{G} tiles x {T2} rows per unit exceed {TPU} threads")
    units = -(-ntiles // G)
    R_unit = G * T2
    cap = (slot_bytes - HDR) // 8
    cap -= cap & 1
    rp = dt.rowptr.cpu().numpy()
    row_len = (rp[:, 1:] - rp[:, :-1])  # (K, n)
    row_tot = row_len.sum(axis=0)
    # virtual threads per row, unit by unit
    m_all = np.empty(n, np.int64)
    vf_list = []
    for u in range(units):
        r0, r1 = u * R_unit, min((u + 1) * R_unit, n)
        m = _threads_per_row(row_tot[r0:r1].astype(np.float64), r1 - r0)
        m_all[r0:r1] = m
        vf = np.zeros(r1 - r0 + 1, np.int64)
        np.cumsum(m, out=vf[1:])
        vf_list.append(vf)
    vstart = np.concatenate([vf[:-1] for vf in vf_list])  # first thread of each row (unit-local)

    # ---- per-entry coordinates on the device
    nnz = dt.nnz
    k_of = torch.repeat_interleave(torch.arange(K, device=dev),
                                   torch.as_tensor(row_len.sum(axis=1), device=dev))
    row_of = torch.repeat_interleave(
        torch.arange(n, device=dev).repeat(K), torch.as_tensor(row_len.reshape(-1), device=dev))
    col = dt.cols.to(torch.int64) & 0xFFFFFFFF
    band = col // BW
    col_local = col % BW
    # position inside the (row, band, k) segment: entries are col-sorted within
    # a row, so segments are contiguous runs
    seg_key = (k_of * n + row_of) * NB + band
    seg_start_flag = torch.ones(nnz, dtype=torch.bool, device=dev)
    seg_start_flag[1:] = seg_key[1:] != seg_key[:-1]
    idx = torch.arange(nnz, device=dev)
    seg_first = torch.cummax(torch.where(seg_start_flag, idx, torch.zeros_like(idx)), 0).values
    pos = idx - seg_first
    seg_len = torch.bincount(torch.cumsum(seg_start_flag.to(torch.int64), 0) - 1)
    seg_len_e = seg_len[torch.cumsum(seg_start_flag.to(torch.int64), 0) - 1]
    m_t = torch.as_tensor(m_all, device=dev)[row_of]
    piece = ((pos + 1) * m_t - 1) // seg_len_e
    thread = torch.as_tensor(vstart, device=dev)[row_of] + piece
    unit = row_of // R_unit
    # stream order: (unit, band, thread, k, col)
    key = ((((unit * NB + band) * TPU + thread) * 16 + k_of) << 16) | col_local
    order = torch.argsort(key)
    unit_s, band_s, thread_s = unit[order], band[order], thread[order]
    ub = unit_s * NB + band_s
    # position inside the (unit, band) group -> sub-item split at `cap`
    grp_flag = torch.ones(nnz, dtype=torch.bool, device=dev)
    grp_flag[1:] = ub[1:] != ub[:-1]
    grp_first = torch.cummax(torch.where(grp_flag, idx, torch.zeros_like(idx)), 0).values
    gpos = idx - grp_first
    sub = gpos // cap
    item_key = ub * 4096 + sub  # (unit, band, sub)
    ik_flag = torch.ones(nnz, dtype=torch.bool, device=dev)
    ik_flag[1:] = item_key[1:] != item_key[:-1]
    item_id = torch.cumsum(ik_flag.to(torch.int64), 0) - 1
    n_items = int(item_id[-1].item()) + 1 if nnz else 0
    item_n = torch.bincount(item_id, minlength=n_items)
    counts = torch.bincount(item_id * TPU + thread_s, minlength=n_items * TPU).view(n_items, TPU)
    if nnz and int(counts.max().item()) > MAXCNT:
        raise ValueError("a virtual thread holds more than 65535 entries of one item")
    first_e = torch.nonzero(ik_flag).squeeze(1)
    item_unit = unit_s[first_e].cpu().numpy()
    item_band = band_s[first_e].cpu().numpy()
    item_n_h = item_n.cpu().numpy().astype(np.int64)
    item_bytes = HDR + 8 * (item_n_h + (item_n_h & 1))
    item_off = np.zeros(n_items + 1, np.int64)
    np.cumsum(item_bytes, out=item_off[1:])
    total = int(item_off[-1])
    # headers
    wb = torch.zeros((n_items, NW + 1), dtype=torch.int64, device=dev)
    wb[:, 1:] = torch.cumsum(counts.view(n_items, NW, 32).sum(dim=2), 1)
    hdr = torch.zeros((n_items, HDR), dtype=torch.uint8, device=dev)
    hdr[:, : 2 * (NW + 1)] = wb.to(torch.int16).view(torch.uint8).view(n_items, 2 * (NW + 1))
    hdr[:, 2 * (NW + 1): 2 * (NW + 1) + 2 * TPU] = (
        counts.to(torch.int32).to(torch.int16).view(torch.uint8).view(n_items, 2 * TPU))
    stream = torch.zeros(total + 16, dtype=torch.uint8, device=dev)[:total]
    off_d = torch.as_tensor(item_off[:-1], device=dev)
    hpos = (off_d[:, None] + torch.arange(HDR, device=dev)[None, :]).reshape(-1)
    stream[hpos] = hdr.reshape(-1)
    # entries: position inside the item = gpos - sub * cap
    ipos = gpos - sub * cap
    dst = (off_d[item_id] + HDR) // 8 + ipos
    vbits = dt.vals.view(torch.int32).to(torch.int64)[order] & 0xFFFFFFFF
    packed = ((k_of[order] << 16) | col_local[order]) | (vbits << 32)
    stream.view(torch.int64)[dst] = packed
    # unit tables
    unit_nitems = np.bincount(item_unit, minlength=units)
    unit_item0 = np.zeros(units, np.int64)
    unit_item0[1:] = np.cumsum(unit_nitems)[:-1]
    items = np.zeros(n_items, ITEM_DTYPE)
    items["off"] = item_off[:-1]
    items["bytes"] = item_bytes
    items["band"] = item_band
    unit_tile0 = np.arange(units) * G
    unit_ntiles = np.minimum(G, ntiles - unit_tile0)
    return V4Layout(
        slot_bytes=slot_bytes, band_width=BW, units=units,
        unit_tile0=torch.as_tensor(unit_tile0.astype(np.int32), device=dev),
        unit_ntiles=torch.as_tensor(unit_ntiles.astype(np.int32), device=dev),
        unit_item0=torch.as_tensor(unit_item0.astype(np.int32), device=dev),
        unit_nitems=torch.as_tensor(unit_nitems.astype(np.int32), device=dev),
        items=torch.as_tensor(items.view(np.uint8), device=dev),
        stream=stream,
        vrow_first=torch.as_tensor(np.concatenate(vf_list).astype(np.uint16).view(np.int16),
                                   device=dev),
        n_items=n_items, stream_bytes=total, header_bytes=HDR * n_items,
        max_unit_items=int(unit_nitems.max()) if units else 0)


def launch_v4(lay: V4Layout, dt, x, g, positions, normals, cam, material, vk, scatter, radiance,
              radiance_unclamped, stream=None):
    _lib.call("sss_transfer_v4", dt.K, dt.side, dt.levels, lay.band_width, lay.slot_bytes,
              lay.units, lay.max_unit_items, _lib.ptr(lay.unit_tile0), _lib.ptr(lay.unit_ntiles),
              _lib.ptr(lay.unit_item0), _lib.ptr(lay.unit_nitems), _lib.ptr(lay.items),
              _lib.ptr(lay.stream), _lib.ptr(lay.vrow_first), _lib.ptr(x), _lib.ptr(g),
              _lib.ptr(positions), _lib.ptr(normals), _lib.ptr(cam), _lib.ptr(material),
              _lib.ptr(vk), _lib.ptr(scatter), _lib.ptr(radiance), _lib.ptr(radiance_unclamped),
              _lib.stream_ptr(stream))
