"""Frame layouts of the compressed transfer operators (path b).

The canonical operator (``transfer.DeviceTransfer``) is one tile-major CSR per
PCA term k: ``rowptr`` (K, N+1) absolute offsets, ``cols`` (tile-major w0 ids,
ascending within a row) and f32 ``vals`` — the reference's
``TransferOperator`` transposed (transfer.py:50-71 stores CSC over w0
columns). The per-frame kernels read copies of it rearranged for the GPU:

* ``kfr_layout`` — the K-fused row-chunk stream of ``sss_transfer_kfr``
  (csrc/transfer.cu, the default): the K terms of a receiver row merged into
  (column, term-mask) pairs, rows cut into chunks of <= ``chunk`` pairs, 32
  chunks per warp item, one pair per lane per step, the f32 values in term
  planes. Built on the device with torch in a few hundred milliseconds.
* ``flat16_layout`` — the flat (row, k)-segment stream of
  ``sss_transfer_flat16`` (csrc/flat16_25.cu), kept as the A/B alternative
  and for operators with more than 65536 rows or 16 terms.

Both are pure data rearrangements: every stored coefficient appears exactly
once (the host tests check both against the CSR product).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

KFR_STEPS_PER_BATCH = 4  # csrc/transfer.cu kKfrU


def _level_class(idx: torch.Tensor, levels: int) -> torch.Tensor:
    """0 for the tile's scaling coefficient, l for detail level l (1 coarsest)
    of a tile-major index (tile * 4^L + local, local in the L-level Mallat
    layout of the tile)."""
    loc = idx % (4 ** levels)
    c = torch.zeros_like(loc)
    for lv in range(1, levels + 1):
        c[(loc >= 4 ** (lv - 1)) & (loc < 4 ** lv)] = lv
    return c


def canonical_entries(t):
    """(row, k, col, val) of every stored coefficient, CSR order (k-major,
    rows ascending, columns ascending)."""
    K, n = t.K, t.n
    dev = t.rowptr.device
    rp = t.rowptr
    lens = rp[:, 1:] - rp[:, :-1]
    k_of = torch.repeat_interleave(torch.arange(K, device=dev), lens.sum(1))
    row_of = torch.repeat_interleave(torch.arange(n, device=dev).repeat(K), lens.reshape(-1))
    lo, hi = int(rp[0, 0]), int(rp[-1, -1])
    col = t.cols[lo:hi].to(torch.int64) & 0xFFFFFFFF
    return row_of, k_of, col, t.vals[lo:hi]


@dataclass
class KfrLayout:
    K: int
    n: int
    n_items: int
    n_partials: int
    items: torch.Tensor      # (n_items, 2) int32 {first batch, steps}
    lane_len: torch.Tensor   # (n_items * 32,) int32
    lane_dst: torch.Tensor   # (n_items * 32,) int32 (u32 bit patterns)
    batch_off: torch.Tensor  # (n_batches + 1, 2) int32 {word, value}
    cm: torch.Tensor         # (n_pairs + pad,) int32: col | mask << 16
    vals: torch.Tensor       # (nnz + pad,) float32, term planes
    partials: torch.Tensor   # (3K, max(n_partials, 1)) float64 scratch
    partial_row: torch.Tensor
    multi_info: torch.Tensor  # (n_multi, 4) int32 {row, first slot, count, 0}
    multi_count: torch.Tensor  # (n_multi,) int32, zero between frames
    stats: dict = field(default_factory=dict)


def _bitrev(mask: torch.Tensor, K: int) -> torch.Tensor:
    r = torch.zeros_like(mask)
    for k in range(K):
        r |= ((mask >> k) & 1) << (K - 1 - k)
    return r


def kfr_layout(t, chunk: int = 512, bucket: int = 16) -> KfrLayout:
    """K-fused row-chunk layout of sss_transfer_kfr (see csrc/transfer.cu).

    Pairs of a row are ordered by term mask (highest terms first: the masks
    of one step across the warp's lanes then share most of their planes),
    then column. Chunks are grouped 32 to a warp item by (row level class,
    length bucket, row) so a warp's lanes have similar lengths (idle lanes
    cost issue slots) and neighbouring rows (coalesced v_k stores); items are
    ordered longest first for the static round-robin assignment."""
    K, n, L = t.K, t.n, t.levels
    if K > 16 or n > 65536:
        raise ValueError("kfr layout: K <= 16 terms and n <= 65536 rows (16-bit columns)")
    dev = t.rowptr.device
    U = KFR_STEPS_PER_BATCH
    row, k, col, val = canonical_entries(t)
    nnz = row.numel()
    key = row * n + col
    o = torch.argsort(key * 16 + k)
    key, k, val = key[o], k[o], val[o]
    del o, row, col
    newp = torch.ones(nnz, dtype=torch.bool, device=dev)
    if nnz:
        newp[1:] = key[1:] != key[:-1]
    pid = torch.cumsum(newp.to(torch.int64), 0) - 1
    P = int(newp.sum())
    pkey = key[newp]
    prow, pcol = pkey // n, pkey % n
    pmask = torch.zeros(P, dtype=torch.int64, device=dev).scatter_add_(
        0, pid, torch.bitwise_left_shift(torch.ones_like(k), k))
    del pkey, newp
    # pair order inside a row: masks with high terms first, then column
    okey = (prow << 33) | (((1 << 16) - 1 - _bitrev(pmask, K)) << 16) | pcol
    po = torch.argsort(okey)
    del okey
    rank_of_pair = torch.empty_like(po)
    rank_of_pair[po] = torch.arange(P, device=dev)
    prow, pcol, pmask = prow[po], pcol[po], pmask[po]
    cnt = torch.bincount(prow, minlength=n)
    start = torch.cumsum(cnt, 0) - cnt
    pos = torch.arange(P, device=dev) - start[prow]
    nch = torch.clamp((cnt + chunk - 1) // chunk, min=1)
    chbase = torch.cumsum(nch, 0) - nch
    pchunk = chbase[prow] + pos // chunk
    pstep = pos % chunk
    NC = int(nch.sum())
    clen = torch.bincount(pchunk, minlength=NC)
    crow = torch.repeat_interleave(torch.arange(n, device=dev), nch)
    cidx = torch.arange(NC, device=dev) - chbase[crow]
    lvl = _level_class(crow, L)
    nb = max(1, (chunk + bucket - 1) // bucket)
    ckey = (lvl << 44) | ((nb - clen // bucket) << 30) | (crow << 12) | cidx
    corder = torch.argsort(ckey)
    NI = (NC + 31) // 32
    slot_len = torch.zeros(NI * 32, dtype=torch.int64, device=dev)
    slot_len[:NC] = clen[corder]
    S = slot_len.view(NI, 32).amax(dim=1)
    iorder = torch.argsort(-S, stable=True)  # longest items first
    inew = torch.empty_like(iorder)
    inew[iorder] = torch.arange(NI, device=dev)
    cpos = torch.empty(NC, dtype=torch.int64, device=dev)
    cpos[corder] = torch.arange(NC, device=dev)
    citem = inew[cpos // 32]
    clane = cpos % 32
    S = S[iorder]
    # partial slots for rows cut into several chunks, consecutive per row
    multi = nch > 1
    mrows = torch.nonzero(multi).flatten()
    M = mrows.numel()
    mcnt = nch[mrows]
    mfirst = torch.cumsum(mcnt, 0) - mcnt
    m_of_row = torch.full((n,), -1, dtype=torch.int64, device=dev)
    m_of_row[mrows] = torch.arange(M, device=dev)
    cm_of = m_of_row[crow]
    n_partials = int(mcnt.sum()) if M else 0
    if M:
        cdst = torch.where(cm_of >= 0, (1 << 31) | (mfirst[cm_of.clamp(min=0)] + cidx), crow)
    else:
        cdst = crow.clone()
    lane_len = torch.zeros(NI * 32, dtype=torch.int64, device=dev)
    lane_dst = torch.full((NI * 32,), 0xFFFFFFFF, dtype=torch.int64, device=dev)
    lane_len[citem * 32 + clane] = clen
    lane_dst[citem * 32 + clane] = cdst
    partial_row = torch.repeat_interleave(torch.arange(M, device=dev), mcnt) if M else \
        torch.zeros(1, dtype=torch.int64, device=dev)
    multi_info = torch.zeros((max(M, 1), 4), dtype=torch.int64, device=dev)
    if M:
        multi_info[:, 0] = mrows
        multi_info[:, 1] = mfirst
        multi_info[:, 2] = mcnt
    # word stream: pairs ordered (item, step, lane)
    item_p = citem[pchunk]
    lane_p = clane[pchunk]
    skey = (item_p << 25) | (pstep << 5) | lane_p
    so = torch.argsort(skey)
    skey_sorted = skey[so]
    cm = (pcol | (pmask << 16))[so]
    # value stream: entries ordered (item, step, term, lane)
    ent_pair = rank_of_pair[pid]  # pair index (new order) of every sorted entry
    vkey = (item_p[ent_pair] << 30) | (pstep[ent_pair] << 14) | (k << 5) | lane_p[ent_pair]
    vo = torch.argsort(vkey)
    vkey_sorted = vkey[vo]
    vals = val[vo]
    del vkey, vo, ent_pair
    # batches of U steps per item: first word / value of step b*U
    nbat = (S + U - 1) // U
    bbase = torch.cumsum(nbat, 0) - nbat
    NB = int(nbat.sum())
    bitem = torch.repeat_interleave(torch.arange(NI, device=dev), nbat)
    bstep = (torch.arange(NB, device=dev) - bbase[bitem]) * U
    q_w = (bitem << 25) | (bstep << 5)
    q_v = (bitem << 30) | (bstep << 14)
    boff = torch.zeros((NB + 1, 2), dtype=torch.int64, device=dev)
    boff[:NB, 0] = torch.searchsorted(skey_sorted, q_w)
    boff[:NB, 1] = torch.searchsorted(vkey_sorted, q_v)
    boff[NB, 0] = P
    boff[NB, 1] = nnz
    items = torch.stack([bbase, S], dim=1)
    pad = 8  # bulk copies round the last batch up to 16 bytes
    cm_t = torch.zeros(P + pad, dtype=torch.int32, device=dev)
    cm_t[:P] = cm.to(torch.int32)
    vals_t = torch.zeros(nnz + pad, dtype=torch.float32, device=dev)
    vals_t[:nnz] = vals

    def u32(x):
        return torch.where(x >= (1 << 31), x - (1 << 32), x).to(torch.int32).contiguous()

    steps = int(S.sum())
    stats = {"pairs": P, "entries": nnz, "chunks": NC, "items": NI, "steps": steps,
             "batches": NB, "lane_util": round(P / max(32 * steps, 1), 4),
             "multi_rows": M, "partials": n_partials,
             "bytes": (P + pad) * 4 + (nnz + pad) * 4 + NI * 8 + NI * 256 + (NB + 1) * 8}
    return KfrLayout(
        K=K, n=n, n_items=NI, n_partials=n_partials, items=u32(items), lane_len=u32(lane_len),
        lane_dst=u32(lane_dst), batch_off=u32(boff), cm=cm_t, vals=vals_t,
        partials=torch.zeros((3 * K, max(n_partials, 1)), dtype=torch.float64, device=dev),
        partial_row=u32(partial_row), multi_info=u32(multi_info),
        multi_count=torch.zeros(max(M, 1), dtype=torch.int32, device=dev), stats=stats)


def kfr_reference_apply(lay: KfrLayout, x: torch.Tensor) -> torch.Tensor:
    """Decode the kfr stream on the host side of torch (any device) and apply
    it: v (K, 3, n) = T_k x_c. For layout tests; mirrors the kernel's
    indexing (compacted words per step, term planes)."""
    K, n = lay.K, lay.n
    dev = lay.cm.device
    items = lay.items.long()
    lane_len = lay.lane_len.long().view(-1, 32)
    dst = lay.lane_dst.long() & 0xFFFFFFFF
    boff = lay.batch_off.long()
    cm = lay.cm.long() & 0xFFFFFFFF
    vals = lay.vals.double()
    v = torch.zeros((K, 3, n), dtype=torch.float64, device=dev)
    part = torch.zeros((3 * K, max(lay.n_partials, 1)), dtype=torch.float64, device=dev)
    x = x.double()
    lanes = torch.arange(32, device=dev)
    for i in range(lay.n_items):
        b0, S = int(items[i, 0]), int(items[i, 1])
        w = int(boff[b0, 0]) if S else 0
        vo = int(boff[b0, 1]) if S else 0
        acc = torch.zeros((32, K, 3), dtype=torch.float64, device=dev)
        for s in range(S):
            act = s < lane_len[i]
            na = int(act.sum())
            words = torch.zeros(32, dtype=torch.int64, device=dev)
            words[act] = cm[w:w + na]
            w += na
            col, mask = words & 0xFFFF, words >> 16
            xs = x[:, col].T  # (32, 3)
            for k in range(K):
                has = ((mask >> k) & 1).bool() & act
                m = int(has.sum())
                if m:
                    acc[has, k, :] += vals[vo:vo + m, None] * xs[has]
                    vo += m
        d = dst[i * 32:(i + 1) * 32]
        for ln in lanes.tolist():
            dd = int(d[ln])
            if dd == 0xFFFFFFFF:
                continue
            if dd & 0x80000000:
                part[:, dd & 0x7FFFFFFF] = acc[ln].reshape(-1)
            else:
                v[:, :, dd] = acc[ln]
    info = lay.multi_info.long()
    for m in range(info.shape[0] if lay.n_partials else 0):
        r, f, c = int(info[m, 0]), int(info[m, 1]), int(info[m, 2])
        v[:, :, r] = part[:, f:f + c].sum(dim=1).view(K, 3)
    return v


def flat16_layout(t, warps_per_sm: int = 32, col16: bool = None):
    """The flat16 stream (csrc/flat16_25.cu): (row, k) segments in row-major
    order, each padded to a multiple of 16 entries (column 0 / value 0, or
    column n with 32-bit columns) and lane-interleaved (entry e * L + j of a
    segment of 16 L entries -> lane j, slot e); head bit per 16-entry group at
    every segment start, per-word head prefix, segment ids row << 4 | k, and
    equal word ranges for `warps_per_sm` warps per SM. Returns the tuple the
    runtime launches with."""
    E = 16
    K, n = t.K, t.n
    dev = t.rowptr.device
    if col16 is None:
        col16 = n <= 65536
    rp = t.rowptr
    lens = (rp[:, 1:] - rp[:, :-1]).T.reshape(-1)  # (row, k) order
    starts = rp[:, :-1].T.reshape(-1)
    rowk = (torch.arange(n, device=dev)[:, None] * 16 + torch.arange(K, device=dev)[None, :]).reshape(-1)
    keep = lens > 0
    lens, starts, rowk = lens[keep], starts[keep], rowk[keep]
    lp = (lens + E - 1) // E * E
    dst = torch.cumsum(lp, 0) - lp
    total = int(lp.sum())
    fill_col = 0 if col16 else n
    pcols = torch.full((max(total, E),), fill_col, dtype=torch.int64, device=dev)
    pvals = torch.zeros(max(total, E), dtype=torch.float32, device=dev)
    seg = torch.repeat_interleave(torch.arange(lens.numel(), device=dev), lens)
    q = torch.arange(seg.numel(), device=dev) - torch.repeat_interleave(torch.cumsum(lens, 0) - lens, lens)
    Lanes = lp[seg] // E
    d = dst[seg] + (q % Lanes) * E + q // Lanes
    src = starts[seg] + q
    pcols[d] = t.cols[src].to(torch.int64) & 0xFFFFFFFF
    pvals[d] = t.vals[src]
    del seg, q, Lanes, d, src
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 8
    ng = pcols.numel() // E
    nw = (ng + 31) // 32
    s4 = dst // E
    heads = torch.zeros(nw, dtype=torch.int64, device=dev).index_add_(
        0, s4 // 32, torch.bitwise_left_shift(torch.ones_like(s4), s4 % 32))
    heads = torch.where(heads >= (1 << 31), heads - (1 << 32), heads).to(torch.int32)
    cnt = torch.bincount(s4 // 32, minlength=nw)
    hpre = (torch.cumsum(cnt, 0) - cnt).to(torch.int32)
    wbeg = (torch.arange(W + 1, dtype=torch.int64, device=dev) * nw) // W
    if col16:
        pc = torch.where(pcols >= 32768, pcols - 65536, pcols).to(torch.int16)
    else:
        pc = pcols.to(torch.int32)
    stats = {"entries": pcols.numel(), "words": nw, "segments": int(s4.numel()),
             "E": E, "col_bits": 16 if col16 else 32}
    return (pc.contiguous(), pvals, pcols.numel(), heads.contiguous(), hpre.contiguous(),
            rowk.to(torch.int32).contiguous(), wbeg.to(torch.int32).contiguous(), W, stats)
