"""Build the frame layout v4 (csrc/stream4.cu) from the canonical tile-major
CSR operator: per-SM units, virtual threads, self-describing (band, k) items.

Host-side planning in numpy (row splits, per-thread counts, item headers,
item table); the 8-byte entries are gathered into the stream on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

NW = 16  # consumer warps (csrc/stream4.cu: kV4Warps)
TPU = NW * 32
SLOTS = 4
HDR = (2 * (NW + 1) + TPU + 15) & ~15  # u16 warp bases + u8 counts, 16-B padded
MAXCNT = 255

ITEM_DTYPE = np.dtype([("off", "<u8"), ("bytes", "<u4"), ("band", "<u2"), ("k", "u1"),
                       ("pad", "u1")])


@dataclass
class V4Layout:
    slot_bytes: int
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
    max_unit_items: int = 0


def _ragged(starts, lens, device):
    """concat(arange(s, s + l)) on the device."""
    starts = torch.as_tensor(starts, dtype=torch.int64, device=device)
    lens = torch.as_tensor(lens, dtype=torch.int64, device=device)
    total = int(lens.sum().item())
    if total == 0:
        return torch.empty(0, dtype=torch.int64, device=device)
    rep_s = torch.repeat_interleave(starts, lens)
    base = torch.repeat_interleave(torch.cumsum(lens, 0) - lens, lens)
    return torch.arange(total, device=device) - base + rep_s


def build_v4(dt, slot_bytes: int = 24576, n_sm: int = None) -> V4Layout:
    dev = dt.rowptr.device
    if n_sm is None:
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    n, K, NB, BW = dt.n, dt.K, dt.n_bands, dt.band_width
    T2 = (1 << dt.levels) ** 2
    ntiles = n // T2
    G = -(-ntiles // n_sm)
    if G * T2 > TPU:
        raise ValueError(f"{G} tiles x {T2} rows per unit exceed {TPU} threads")
    units = -(-ntiles // G)
    cap = (slot_bytes - HDR) // 8
    cap -= cap & 1
    rp = dt.rowptr.cpu().numpy()
    bo = dt.bandoff.cpu().numpy().astype(np.int64)  # (K, n, NB+1)
    seg_len_all = np.diff(bo, axis=2)  # (K, n, NB)
    row_tot = seg_len_all.sum(axis=(0, 2))

    item_recs, item_hdrs, item_n = [], [], []
    seg_starts, seg_lens = [], []
    unit_tile0, unit_ntiles, unit_item0, unit_nitems, vrow_first = [], [], [], [], []
    for u in range(units):
        t0 = u * G
        nt = min(G, ntiles - t0)
        r0, R = t0 * T2, nt * T2
        rows = np.arange(r0, r0 + R)
        # virtual threads: 1 per row + the spare ones proportional to length
        Lr = row_tot[rows].astype(np.float64)
        spare = TPU - R
        m = np.ones(R, np.int64)
        if spare > 0 and Lr.sum() > 0:
            share = spare * Lr / Lr.sum()
            extra = np.floor(share).astype(np.int64)
            rem = spare - int(extra.sum())
            if rem > 0:
                extra[np.argsort(-(share - extra), kind="stable")[:rem]] += 1
            m += extra
        vf = np.zeros(R + 1, np.int64)
        np.cumsum(m, out=vf[1:])
        nthreads_used = int(vf[-1])
        thr_row = np.repeat(np.arange(R), m)  # row of each virtual thread
        thr_j = np.arange(nthreads_used) - vf[thr_row]
        thr_m = m[thr_row]
        unit_tile0.append(t0)
        unit_ntiles.append(nt)
        unit_item0.append(len(item_recs))
        vrow_first.append(vf.astype(np.uint16))
        lens = seg_len_all[:, rows, :]  # (K, R, NB)
        starts = rp[:, rows][:, :, None] + bo[:, rows, :NB]  # (K, R, NB)
        for b in range(NB):
            for k in range(K):
                ln = lens[k, :, b]
                ntot = int(ln.sum())
                if ntot == 0:
                    continue
                lt = ln[thr_row]
                cnt = (lt * (thr_j + 1)) // thr_m - (lt * thr_j) // thr_m
                counts = np.zeros(TPU, np.int64)
                counts[:nthreads_used] = cnt
                seg_starts.append(starts[k, :, b])
                seg_lens.append(ln)
                for sub in _split(counts, cap):
                    hdr = np.zeros(HDR, np.uint8)
                    wb = np.zeros(NW + 1, np.int64)
                    np.cumsum(sub.reshape(NW, 32).sum(axis=1), out=wb[1:])
                    hdr[: 2 * (NW + 1)] = wb.astype("<u2").view(np.uint8)
                    hdr[2 * (NW + 1): 2 * (NW + 1) + TPU] = sub.astype(np.uint8)
                    ns = int(sub.sum())
                    item_hdrs.append(hdr)
                    item_n.append(ns)
                    item_recs.append((b, k))
        unit_nitems.append(len(item_recs) - unit_item0[-1])

    n_items = len(item_recs)
    item_n = np.asarray(item_n, np.int64)
    item_bytes = HDR + 8 * (item_n + (item_n & 1))
    item_off = np.zeros(n_items + 1, np.int64)
    np.cumsum(item_bytes, out=item_off[1:])
    total = int(item_off[-1])
    items = np.zeros(n_items, ITEM_DTYPE)
    items["off"] = item_off[:-1]
    items["bytes"] = item_bytes
    items["band"] = [b for b, _ in item_recs]
    items["k"] = [k for _, k in item_recs]
    # stream: headers on the host, entries gathered on the device
    host = np.zeros(total, np.uint8)
    hdr_pos = _ragged_np(item_off[:-1], np.full(n_items, HDR))
    host[hdr_pos] = np.concatenate(item_hdrs) if item_hdrs else np.empty(0, np.uint8)
    stream = torch.as_tensor(host, device=dev)
    src = _ragged(np.concatenate(seg_starts), np.concatenate(seg_lens), dev)
    dst = _ragged((item_off[:-1] + HDR) // 8, item_n, dev)
    cols = dt.cols[src].to(torch.int64) & 0xFFFFFFFF
    vbits = dt.vals[src].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    packed = (cols % BW) | (vbits << 32)
    stream.view(torch.int64)[dst] = packed
    return V4Layout(
        slot_bytes=slot_bytes, units=units,
        unit_tile0=torch.as_tensor(np.asarray(unit_tile0, np.int32), device=dev),
        unit_ntiles=torch.as_tensor(np.asarray(unit_ntiles, np.int32), device=dev),
        unit_item0=torch.as_tensor(np.asarray(unit_item0, np.int32), device=dev),
        unit_nitems=torch.as_tensor(np.asarray(unit_nitems, np.int32), device=dev),
        items=torch.as_tensor(items.view(np.uint8), device=dev),
        stream=stream,
        vrow_first=torch.as_tensor(np.concatenate(vrow_first).view(np.int16), device=dev),
        n_items=n_items, stream_bytes=total, header_bytes=HDR * n_items,
        max_unit_items=int(max(unit_nitems)) if unit_nitems else 0)


def _ragged_np(starts, lens):
    starts = np.asarray(starts, np.int64)
    lens = np.asarray(lens, np.int64)
    total = int(lens.sum())
    base = np.repeat(np.cumsum(lens) - lens, lens)
    return np.arange(total, dtype=np.int64) - base + np.repeat(starts, lens)


def _split(counts, cap):
    """Cut one item's per-thread counts into sub-items with <= cap entries and
    <= 255 entries per thread; entry order is preserved."""
    if counts.sum() <= cap and counts.max() <= MAXCNT:
        return [counts]
    out, cur, cur_n = [], np.zeros_like(counts), 0
    for t in range(counts.size):
        r = int(counts[t])
        while r > 0:
            take = min(r, MAXCNT - int(cur[t]), cap - cur_n)
            if take <= 0:
                out.append(cur)
                cur, cur_n = np.zeros_like(counts), 0
                continue
            cur[t] += take
            cur_n += take
            r -= take
            if cur_n == cap:
                out.append(cur)
                cur, cur_n = np.zeros_like(counts), 0
    if cur_n:
        out.append(cur)
    return out


def launch_v4(lay: V4Layout, dt, x, g, positions, normals, cam, material, vk, scatter, radiance,
              radiance_unclamped, stream=None):
    _lib.call("sss_transfer_v4", dt.K, dt.side, dt.levels, dt.band_width, lay.slot_bytes,
              lay.units, lay.max_unit_items, _lib.ptr(lay.unit_tile0), _lib.ptr(lay.unit_ntiles),
              _lib.ptr(lay.unit_item0), _lib.ptr(lay.unit_nitems), _lib.ptr(lay.items),
              _lib.ptr(lay.stream), _lib.ptr(lay.vrow_first), _lib.ptr(x), _lib.ptr(g),
              _lib.ptr(positions), _lib.ptr(normals), _lib.ptr(cam), _lib.ptr(material),
              _lib.ptr(vk), _lib.ptr(scatter), _lib.ptr(radiance), _lib.ptr(radiance_unclamped),
              _lib.stream_ptr(stream))
