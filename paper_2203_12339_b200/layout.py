"""Frame layouts of the compressed transfer operators (path b).

The canonical operator (``transfer.DeviceTransfer``) is one tile-major CSR per
PCA term k: ``rowptr`` (K, N+1) absolute offsets, ``cols`` (tile-major w0 ids,
ascending within a row) and f32 ``vals`` — the reference's
``TransferOperator`` transposed (transfer.py:50-71 stores CSC over w0
columns). The per-frame kernels read copies of it rearranged for the GPU:

* ``kfr_layout`` — the K-fused row-chunk stream of ``sss_transfer_kfr``
  (csrc/transfer.cu, the default): the terms of a receiver row merged, in
  groups of 4, into (column, term-mask) pairs, (row, group)s cut into chunks
  of <= ``chunk`` pairs, 32 chunks per warp item, one pair per lane per step.
  Built on the device with torch in well under a second.
* ``flat16_layout`` — the flat (row, k)-segment stream of
  ``sss_transfer_flat16`` (csrc/flat16_25.cu), kept as the A/B alternative
  and for operators with more than 65536 rows or 16 terms.

Both are pure data rearrangements: every stored coefficient appears exactly
once (the host tests check both against the CSR product).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

KFR_GROUP = 4  # csrc/transfer.cu kKfrG: terms accumulated per chunk
KFR_MAX_BATCHES = 128  # csrc/transfer.cu kKfrMaxBatches


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
    lane_len: torch.Tensor   # (n_items * 32,) int32 chunk lengths (pairs)
    lane_dst: torch.Tensor   # (n_items * 32,) int32: row | group << 16, 1 << 31 | slot, or -1
    batch_off: torch.Tensor  # (n_batches + 1,) int32 (u32) byte offsets into stream
    stream: torch.Tensor     # int32 words: per batch U * 32 pair words, then f32 values
    partials: torch.Tensor   # (3 G, max(n_partials, 1)) float64 scratch
    partial_row: torch.Tensor
    multi_info: torch.Tensor  # (n_multi, 4) int32 {row, first slot, count, group}
    multi_count: torch.Tensor  # (n_multi,) int32, zero between frames
    work: torch.Tensor = None  # (2,) int32 claim / exit counters, zero between frames
    stats: dict = field(default_factory=dict)


def _bitrev(mask: torch.Tensor, K: int) -> torch.Tensor:
    r = torch.zeros_like(mask)
    for k in range(K):
        r |= ((mask >> k) & 1) << (K - 1 - k)
    return r


def kfr_auto_chunk(n_pairs: int, n_warps: int, steps_per_batch: int) -> int:
    """Chunk length for an operator of `n_pairs` (column, mask) pairs streamed
    by `n_warps` resident warps. A warp item is 32 chunks, so the longest item
    is at most `chunk` steps: measured on the C3 operator, time is lowest while
    that stays just under the mean work per warp (steps / warps: 423 at 2
    CTAs/SM, optimum 376-400 with long rows cut into equal chunks; 282 at 3,
    optimum 272) - longer and the longest item is the makespan, shorter and
    rows split into more partial sums than needed
    (profiles/r02_transfer_experiments.json, chunk sweeps)."""
    steps = n_pairs / 32.0 / 0.974  # the layouts fill ~97.4 % of the lane slots
    U = steps_per_batch
    c = int(0.93 * steps / max(n_warps, 1)) // U * U
    return max(64, min(c, KFR_MAX_BATCHES * U))


def kfr_layout(t, chunk: int = 256, bucket: int = 16, steps_per_batch: int = 4,
               n_warps: int = 0) -> KfrLayout:
    """K-fused row-chunk layout of sss_transfer_kfr (see csrc/transfer.cu).

    The K terms are split in groups of G = KFR_GROUP; the terms of one
    (receiver row, group) merge into (column, G-bit term mask) pairs, ordered
    by mask (highest terms first) then column and cut into chunks of <=
    `chunk` pairs (every (row, group) has at least one, possibly empty,
    chunk: its v_k rows are written even when zero). A warp item is 32
    chunks, one per lane; step s of an item holds the s-th pair of every
    lane: 32 dense words {col | mask << 16 | offset << 20} (0 where the lane's
    chunk has ended) and the lanes' values lane-major (offset = the lane's
    first value in the batch's value block). Chunks are grouped by (row level class, length
    bucket, row, group) so an item's lanes have similar lengths and
    neighbouring rows; items are ordered longest first (dynamic claiming)."""
    G = KFR_GROUP
    K, n, L = t.K, t.n, t.levels
    NG = (K + G - 1) // G
    if K > 4 * G or n > 65536:
        raise ValueError("kfr layout: K <= 16 terms and n <= 65536 rows (16-bit columns)")
    if chunk > KFR_MAX_BATCHES * steps_per_batch:
        raise ValueError(f"kfr layout: chunk <= {KFR_MAX_BATCHES} x steps_per_batch")
    auto_chunk = chunk <= 0  # chosen below from the pair count and `n_warps`
    dev = t.rowptr.device
    U = steps_per_batch
    row, k, col, val = canonical_entries(t)
    nnz = row.numel()
    grp, kl = k // G, k % G
    key = (row * NG + grp) * n + col
    o = torch.argsort(key * G + kl)
    key, kl, val = key[o], kl[o], val[o]
    del o, row, col, k, grp
    newp = torch.ones(nnz, dtype=torch.bool, device=dev)
    if nnz:
        newp[1:] = key[1:] != key[:-1]
    pid = torch.cumsum(newp.to(torch.int64), 0) - 1
    P = int(newp.sum())
    pkey = key[newp]
    prg, pcol = pkey // n, pkey % n  # prg = row * NG + group
    pmask = torch.zeros(P, dtype=torch.int64, device=dev).scatter_add_(
        0, pid, torch.bitwise_left_shift(torch.ones_like(kl), kl))
    del pkey, newp, key
    # pair order inside a (row, group): masks with high terms first, then column
    okey = (prg << 24) | (((1 << G) - 1 - _bitrev(pmask, G)) << 16) | pcol
    po = torch.argsort(okey)
    del okey
    rank_of_pair = torch.empty_like(po)
    rank_of_pair[po] = torch.arange(P, device=dev)
    prg, pcol, pmask = prg[po], pcol[po], pmask[po]
    if auto_chunk:
        chunk = kfr_auto_chunk(P, n_warps, U)
    RG = n * NG
    cnt = torch.bincount(prg, minlength=RG)
    start = torch.cumsum(cnt, 0) - cnt
    pos = torch.arange(P, device=dev) - start[prg]
    nch = torch.clamp((cnt + chunk - 1) // chunk, min=1)
    chbase = torch.cumsum(nch, 0) - nch
    # a (row, group) longer than `chunk` is cut into equal chunks (420 pairs at
    # chunk 408 -> 210 + 210, not 408 + 12): shorter longest items for the
    # same number of partial sums (142.6 -> 137.9 us on the C3 operator)
    cs = torch.clamp((cnt + nch - 1) // nch, min=1)
    pchunk = chbase[prg] + pos // cs[prg]
    pstep = pos % cs[prg]
    NC = int(nch.sum())
    clen = torch.bincount(pchunk, minlength=NC)
    crg = torch.repeat_interleave(torch.arange(RG, device=dev), nch)
    crow, cgrp = crg // NG, crg % NG
    cidx = torch.arange(NC, device=dev) - chbase[crg]
    lvl = _level_class(crow, L)
    nb = max(1, (chunk + bucket - 1) // bucket)
    ckey = (lvl << 48) | ((nb - clen // bucket) << 36) | (crow << 20) | (cgrp << 16) | cidx
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
    # partial slots for (row, group)s cut into several chunks, consecutive
    multi = nch > 1
    mrg = torch.nonzero(multi).flatten()
    M = mrg.numel()
    mcnt = nch[mrg]
    mfirst = torch.cumsum(mcnt, 0) - mcnt
    m_of = torch.full((RG,), -1, dtype=torch.int64, device=dev)
    m_of[mrg] = torch.arange(M, device=dev)
    cm_of = m_of[crg]
    n_partials = int(mcnt.sum()) if M else 0
    direct = crow | (cgrp << 16)
    if M:
        cdst = torch.where(cm_of >= 0, (1 << 31) | (mfirst[cm_of.clamp(min=0)] + cidx), direct)
    else:
        cdst = direct
    lane_len = torch.zeros(NI * 32, dtype=torch.int64, device=dev)
    lane_dst = torch.full((NI * 32,), 0xFFFFFFFF, dtype=torch.int64, device=dev)
    lane_len[citem * 32 + clane] = clen
    lane_dst[citem * 32 + clane] = cdst
    partial_row = torch.repeat_interleave(torch.arange(M, device=dev), mcnt) if M else \
        torch.zeros(1, dtype=torch.int64, device=dev)
    multi_info = torch.zeros((max(M, 1), 4), dtype=torch.int64, device=dev)
    if M:
        multi_info[:, 0] = mrg // NG
        multi_info[:, 1] = mfirst
        multi_info[:, 2] = mcnt
        multi_info[:, 3] = mrg % NG
    # batches of U steps per item; batch = [U * 32 words | values], 16-byte padded
    item_p = citem[pchunk]
    lane_p = clane[pchunk]
    nbat = (S + U - 1) // U
    bbase = torch.cumsum(nbat, 0) - nbat
    NB = int(nbat.sum())
    pbatch = bbase[item_p] + pstep // U
    # values ordered (item, step, lane, term) = (batch, step, lane, term)
    ent_pair = rank_of_pair[pid]
    vkey = (item_p[ent_pair] << 30) | (pstep[ent_pair] << 14) | (lane_p[ent_pair] << 4) | kl
    vo = torch.argsort(vkey)
    vkey_sorted = vkey[vo]
    vals = val[vo]
    vpos = torch.empty(nnz, dtype=torch.int64, device=dev)
    vpos[vo] = torch.arange(nnz, device=dev)
    del vkey, vo
    # first value of every pair, of every step and of every batch (global order)
    pfirst = torch.full((P,), nnz, dtype=torch.int64, device=dev).scatter_reduce_(
        0, ent_pair, vpos, "amin")
    bitem = torch.repeat_interleave(torch.arange(NI, device=dev), nbat)
    bstep = (torch.arange(NB, device=dev) - bbase[bitem]) * U
    bv0 = torch.searchsorted(vkey_sorted, (bitem << 30) | (bstep << 14))
    # the pair's first value, counted from the start of its BATCH's value block
    # (<= U * 32 * G values: 12 bits at 8 steps): no running per-step base in
    # the kernel, so the value loads of a batch's steps do not wait on one
    # another
    poff = pfirst - bv0[pbatch]
    if P and int(poff.max()) >= 4096:
        raise AssertionError("kfr layout: batch value offset overflow")
    bv1 = torch.cat([bv0[1:], torch.tensor([nnz], device=dev)]) if NB else bv0
    bwords = (U * 32 * 4) // 4
    bsize = bwords + ((bv1 - bv0) + 3) // 4 * 4  # in 4-byte units, 16-byte multiples
    bstart = torch.cumsum(bsize, 0) - bsize
    total = int(bsize.sum()) if NB else 0
    stream = torch.zeros(total + 4, dtype=torch.int32, device=dev)
    wv = (pcol | (pmask << 16) | (poff << 20)).to(torch.int64)
    wv = torch.where(wv >= (1 << 31), wv - (1 << 32), wv).to(torch.int32)
    stream[bstart[pbatch] + (pstep % U) * 32 + lane_p] = wv
    vb = bbase[item_p[ent_pair]] + pstep[ent_pair] // U  # batch of every entry
    stream[bstart[vb] + bwords + (vpos - bv0[vb])] = val.view(torch.int32)
    del ent_pair, vpos, vb, wv
    boff = torch.zeros(NB + 1, dtype=torch.int64, device=dev)
    boff[:NB] = bstart * 4
    boff[NB] = total * 4
    if total * 4 >= (1 << 32):
        raise ValueError("kfr layout: stream larger than 4 GB")
    items = torch.stack([bbase, S], dim=1)

    def u32(x):
        return torch.where(x >= (1 << 31), x - (1 << 32), x).to(torch.int32).contiguous()

    steps = int(S.sum())
    stats = {"steps_per_batch": U, "chunk": chunk, "groups": NG, "pairs": P, "entries": nnz, "chunks": NC,
             "items": NI, "steps": steps, "batches": NB,
             "lane_util": round(P / max(32 * steps, 1), 4), "multi": M, "partials": n_partials,
             "bytes": total * 4 + NI * 8 + NI * 256 + (NB + 1) * 4}
    return KfrLayout(
        K=K, n=n, n_items=NI, n_partials=n_partials, items=u32(items), lane_len=u32(lane_len),
        lane_dst=u32(lane_dst), batch_off=u32(boff), stream=stream,
        partials=torch.zeros((3 * G, max(n_partials, 1)), dtype=torch.float64, device=dev),
        partial_row=u32(partial_row), multi_info=u32(multi_info),
        multi_count=torch.zeros(max(M, 1), dtype=torch.int32, device=dev),
        work=torch.zeros(2, dtype=torch.int32, device=dev), stats=stats)


def kfr_reference_apply(lay: KfrLayout, x: torch.Tensor) -> torch.Tensor:
    """Decode the kfr stream with torch (any device) and apply it: v (K, 3, n)
    = T_k x_c. For layout tests; mirrors the kernel's indexing (per batch U x
    32 words then the values, lane-major per step at the word's offset,
    partial sums of long (row, group)s summed in chunk order)."""
    G = KFR_GROUP
    K, n = lay.K, lay.n
    dev = lay.stream.device
    items = lay.items.long()
    dst = lay.lane_dst.long() & 0xFFFFFFFF
    boff = lay.batch_off.long() & 0xFFFFFFFF
    words = lay.stream.long() & 0xFFFFFFFF
    vals = lay.stream.view(torch.float32).double()
    v = torch.zeros((K, 3, n), dtype=torch.float64, device=dev)
    part = torch.zeros((3 * G, max(lay.n_partials, 1)), dtype=torch.float64, device=dev)
    x = x.double()
    U = lay.stats["steps_per_batch"]
    for i in range(lay.n_items):
        b0, S = int(items[i, 0]), int(items[i, 1])
        acc = torch.zeros((32, G, 3), dtype=torch.float64, device=dev)
        for s in range(S):
            b = b0 + s // U
            base = int(boff[b]) // 4
            w = words[base + (s % U) * 32: base + (s % U) * 32 + 32]
            vbase = base + U * 32  # offsets count from the batch's value block
            col, mask, off = w & 0xFFFF, (w >> 16) & 0xF, (w >> 20) & 0xFFF
            xs = x[:, col].T  # (32, 3)
            for ln in range(32):
                a = vbase + int(off[ln])
                for k in range(G):
                    if (int(mask[ln]) >> k) & 1:
                        acc[ln, k] += vals[a] * xs[ln]
                        a += 1
        for ln in range(32):
            dd = int(dst[i * 32 + ln])
            if dd == 0xFFFFFFFF:
                continue
            if dd & 0x80000000:
                part[:, dd & 0x7FFFFFFF] = acc[ln].reshape(-1)
            else:
                row, k0 = dd & 0xFFFF, (dd >> 16) * G
                for k in range(G):
                    if k0 + k < K:
                        v[k0 + k, :, row] = acc[ln, k]
    info = lay.multi_info.long()
    for m in range(info.shape[0] if lay.n_partials else 0):
        r, f, c, g = (int(z) for z in info[m])
        s = part[:, f:f + c].sum(dim=1).view(G, 3)
        for k in range(G):
            if g * G + k < K:
                v[g * G + k, :, r] = s[k]
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
    # for the deterministic merge: the word in which the row running into word
    # b began = the last word before b that holds a head
    has = (cnt > 0).to(torch.int64) * torch.arange(nw, device=dev)
    last_head = torch.cummax(has, 0).values
    span_first = torch.zeros(nw, dtype=torch.int64, device=dev)
    span_first[1:] = last_head[:-1]
    stats = {"entries": pcols.numel(), "words": nw, "segments": int(s4.numel()),
             "E": E, "col_bits": 16 if col16 else 32,
             "span_first": span_first.to(torch.int32).contiguous()}
    return (pc.contiguous(), pvals, pcols.numel(), heads.contiguous(), hpre.contiguous(),
            rowk.to(torch.int32).contiguous(), wbeg.to(torch.int32).contiguous(), W, stats)
