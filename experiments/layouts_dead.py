"""Layout builders of the abandoned transfer variants (moved out of
runtime.py; not imported by the product)."""
# flake8: noqa
def csr7_schedule(t: DeviceTransfer, rows_per_cta: int = None):
    """Per-CTA longest-first (row, k) work lists for sss_transfer_csr7."""
    if rows_per_cta is None:
        import os

        rows_per_cta = int(os.environ.get("SSS_CSR7_ROWS", "64"))
    T2 = (1 << t.levels) ** 2
    ntiles = t.n // T2
    G = max(1, min(ntiles, rows_per_cta // T2))
    while ntiles % G:
        G -= 1
    R = G * T2
    rp = t.rowptr.cpu().numpy()
    seg = (rp[:, 1:] - rp[:, :-1]).T  # (n, K) segment lengths
    ctas = ntiles // G
    order = np.empty((ctas, R * t.K), np.uint16)
    for c in range(ctas):
        lens = seg[c * R:(c + 1) * R].reshape(-1)  # index = row_local * K + k
        o = np.argsort(-lens, kind="stable")
        order[c] = ((o // t.K) << 4) | (o % t.K)
    return G, torch.as_tensor(order.view(np.int16), device=t.rowptr.device)


def csr8_schedule(t: DeviceTransfer, split: int = None, warps_per_sm: int = None):
    """(row, k)-ordered segment pieces cut into entry-balanced contiguous
    per-warp ranges for sss_transfer_csr8."""
    import os

    split = split or int(os.environ.get("SSS_CSR8_SPLIT", "2048"))
    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_CSR8_WPS", "48"))
    dev = t.rowptr.device
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    W = nsm * warps_per_sm
    W -= W % 8
    rp = t.rowptr.cpu().numpy()
    starts = rp[:, :-1].T.reshape(-1)  # (row, k) order
    lens = (rp[:, 1:] - rp[:, :-1]).T.reshape(-1)
    rowk = (np.arange(t.n)[:, None] * 16 + np.arange(t.K)[None, :]).reshape(-1)
    keep = lens > 0
    starts, lens, rowk = starts[keep], lens[keep], rowk[keep]
    npc = (lens + split - 1) // split
    rep = np.repeat(np.arange(lens.size), npc)
    j = np.arange(rep.size) - np.repeat(np.cumsum(npc) - npc, npc)
    p_start = starts[rep] + j * split
    p_len = np.minimum(split, lens[rep] - j * split)
    p_rowk = rowk[rep]
    cum = np.concatenate([[0], np.cumsum(p_len)])
    targets = np.arange(W + 1) * (cum[-1] / W)
    wbeg = np.searchsorted(cum, targets, side="left").astype(np.uint32)
    wbeg[-1] = p_len.size
    pieces = np.zeros((p_len.size, 4), np.uint32)
    pieces[:, 0] = p_start
    pieces[:, 1] = p_len
    pieces[:, 2] = p_rowk
    return (torch.as_tensor(pieces.view(np.int32), device=dev),
            torch.as_tensor(wbeg.view(np.int32), device=dev), W)


def csr9_layout(t: DeviceTransfer, split: int = None, warps_per_sm: int = None, pad: int = 4):
    """Padded (multiple-of-4) segment copy + balanced per-warp piece ranges for
    sss_transfer_csr9. Pieces follow (row, k) order (x locality)."""
    import os

    split = split or int(os.environ.get("SSS_CSR9_SPLIT", "1024"))
    split -= split % pad
    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_CSR9_WPS", "32"))
    dev = t.rowptr.device
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 8
    rp = t.rowptr.cpu().numpy()
    starts = rp[:, :-1].T.reshape(-1)  # (row, k) order
    lens = (rp[:, 1:] - rp[:, :-1]).T.reshape(-1)
    rowk = (np.arange(t.n)[:, None] * 16 + np.arange(t.K)[None, :]).reshape(-1)
    keep = lens > 0
    starts, lens, rowk = starts[keep], lens[keep], rowk[keep]
    lens4 = (lens + pad - 1) // pad * pad
    dst = np.zeros(lens.size, np.int64)
    np.cumsum(lens4[:-1], out=dst[1:])
    total = int(lens4.sum())
    # zero-filled: k_pad_segments pads each segment to 4 entries; larger pads
    # (and the tail) must read as column 0, value 0
    pcols = torch.zeros(max(total, pad), dtype=torch.int32, device=dev)
    pvals = torch.zeros(max(total, pad), dtype=torch.float32, device=dev)
    # keep the staging tensors referenced until the kernel has consumed them
    # (a temporary freed before launch can be recycled by the next allocation)
    if dev.type == "cuda":
        d_src = torch.as_tensor(starts.astype(np.int64), device=dev)
        d_len = torch.as_tensor(lens.astype(np.int32), device=dev)
        d_dst = torch.as_tensor(dst, device=dev)
        _lib.call("sss_pad_segments", _lib.ptr(d_src), _lib.ptr(d_len), _lib.ptr(d_dst),
                  int(lens.size), _lib.ptr(t.cols), _lib.ptr(t.vals), _lib.ptr(pcols),
                  _lib.ptr(pvals), _lib.stream_ptr())
        torch.cuda.synchronize()
        del d_src, d_len, d_dst
    else:  # host layout tests
        pcols.zero_()
        pvals.zero_()
        seg = np.repeat(np.arange(lens.size), lens)
        j = np.arange(seg.size) - np.repeat(np.cumsum(lens) - lens, lens)
        src = torch.as_tensor(starts[seg] + j)
        dsti = torch.as_tensor(dst[seg] + j)
        pcols[dsti] = t.cols[src]
        pvals[dsti] = t.vals[src]
    npc = (lens4 + split - 1) // split
    rep = np.repeat(np.arange(lens4.size), npc)
    j = np.arange(rep.size) - np.repeat(np.cumsum(npc) - npc, npc)
    p_start = dst[rep] + j * split
    p_len = np.minimum(split, lens4[rep] - j * split)
    cum = np.concatenate([[0], np.cumsum(p_len)])
    targets = np.arange(W + 1) * (cum[-1] / W)
    wbeg = np.searchsorted(cum, targets, side="left").astype(np.uint32)
    wbeg[-1] = p_len.size
    pieces = np.zeros((p_len.size, 4), np.uint32)
    pieces[:, 0] = p_start
    pieces[:, 1] = p_len
    pieces[:, 2] = rowk[rep]
    return (pcols, pvals, torch.as_tensor(pieces.view(np.int32), device=dev),
            torch.as_tensor(wbeg.view(np.int32), device=dev), W)


def kpack_layout(t: DeviceTransfer, split: int = None, warps_per_sm: int = None):
    """K-packed pair layout + balanced per-warp piece ranges for
    sss_transfer_kpack (built on the device). Every (row, column) pair of the
    K operators is stored once: meta = col | mask << 24, then the f32 values
    of the terms in the mask, k ascending."""
    import os

    split = split or int(os.environ.get("SSS_KPACK_SPLIT", "512"))
    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_KPACK_WPS", "16"))
    if t.K > 8 or t.n > (1 << 24):
        raise ValueError("kpack layout needs K <= 8 and N <= 2^24")
    dev = t.rowptr.device
    n, K = t.n, t.K
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    W = nsm * warps_per_sm
    W -= W % 8
    rp = t.rowptr.to(torch.int64)
    lens = (rp[:, 1:] - rp[:, :-1]).reshape(-1)  # (k, row) order, matches entry order
    kr = torch.arange(K * n, device=dev, dtype=torch.int64)
    # entries of one k are contiguous from rp[k, 0]; the arrays are k-major
    base = int(rp[0, 0].item())
    total = int(lens.sum().item())
    row_of = torch.repeat_interleave(kr % n, lens)
    k_of = torch.repeat_interleave(kr // n, lens)
    col = t.cols[base:base + total].to(torch.int64) & 0xFFFFFFFF
    key = ((row_of * n + col) << 4) | k_of
    key, order = torch.sort(key)
    vals = t.vals[base:base + total][order].contiguous()
    del order, row_of, k_of, col
    pair = key >> 4
    kbit = torch.bitwise_left_shift(torch.ones_like(key), key & 15)
    del key
    upair, inv = torch.unique_consecutive(pair, return_inverse=True)
    del pair
    mask = torch.zeros(upair.numel(), dtype=torch.int64, device=dev)
    mask.index_add_(0, inv, kbit)  # distinct bits: sum == OR
    del kbit, inv
    prow = upair // n
    pcol = upair % n
    meta = pcol | (mask << 24)
    meta = torch.where(meta >= (1 << 31), meta - (1 << 32), meta).to(torch.int32).contiguous()
    cnt = torch.zeros_like(mask)
    for k in range(K):
        cnt += (mask >> k) & 1
    npairs = upair.numel()
    vstart = torch.cumsum(cnt, 0) - cnt  # first value of each pair
    rowcnt = torch.bincount(prow, minlength=n)  # pairs per row
    rowstart = torch.cumsum(rowcnt, 0) - rowcnt
    # rows padded to a multiple of 4 pairs (meta 0 = empty) for 16-byte loads
    rowpad = (rowcnt + 3) // 4 * 4
    padstart = torch.cumsum(rowpad, 0) - rowpad
    npad = int(rowpad.sum().item())
    meta_p = torch.zeros(max(npad, 4), dtype=torch.int32, device=dev)
    meta_p[torch.arange(npairs, device=dev) - rowstart[prow] + padstart[prow]] = meta
    del upair, pcol, mask, prow, meta
    # pieces: rows split into runs of <= split (padded) pairs
    npc = (rowcnt + split - 1) // split
    rows = torch.arange(n, device=dev, dtype=torch.int64)
    rep = torch.repeat_interleave(rows, npc)
    first = torch.cumsum(npc, 0) - npc
    j = torch.arange(rep.numel(), device=dev, dtype=torch.int64) - first[rep]
    p0 = padstart[rep] + j * split
    pn = torch.minimum(torch.full_like(p0, split), rowpad[rep] - j * split)
    u0 = rowstart[rep] + j * split  # first real pair of the piece
    un = torch.minimum(torch.full_like(u0, split), rowcnt[rep] - j * split)
    v0 = vstart[u0]
    vend = torch.where(u0 + un < npairs, vstart[torch.clamp(u0 + un, max=npairs - 1)],
                       torch.full_like(u0, total))
    cost = pn + (vend - v0)  # meta + value loads
    cum = torch.cat([torch.zeros(1, device=dev, dtype=torch.int64), torch.cumsum(cost, 0)])
    targets = (torch.arange(W + 1, device=dev, dtype=torch.float64) * (float(cum[-1]) / W))
    wbeg = torch.searchsorted(cum.to(torch.float64), targets, side="left")
    wbeg[-1] = p0.numel()
    pieces = torch.stack([p0, pn, v0, rep], 1).to(torch.int32).contiguous()
    return (meta_p, vals, pieces, wbeg.to(torch.int32).contiguous(), W, npairs)


def _kpacked_pairs(t: DeviceTransfer):
    """(row, column) pairs of the K operators in (row, column) order: meta =
    column | k-mask << 24 (int64), the values sorted by (row, column, k), the
    pair count per row and each pair's first value."""
    if t.K > 8 or t.n > (1 << 24):
        raise ValueError("K-packed layouts need K <= 8 and N <= 2^24")
    dev = t.rowptr.device
    n, K = t.n, t.K
    i64 = dict(dtype=torch.int64, device=dev)
    rp = t.rowptr.to(torch.int64)
    lens = (rp[:, 1:] - rp[:, :-1]).reshape(-1)
    base = int(rp[0, 0].item())
    total = int(lens.sum().item())
    kr = torch.arange(K * n, **i64)
    row_of = torch.repeat_interleave(kr % n, lens)
    k_of = torch.repeat_interleave(kr // n, lens)
    col = t.cols[base:base + total].to(torch.int64) & 0xFFFFFFFF
    key = ((row_of * n + col) << 4) | k_of
    del row_of, k_of, col
    key, order = torch.sort(key)
    vals = t.vals[base:base + total][order].contiguous()
    del order
    upair, inv = torch.unique_consecutive(key >> 4, return_inverse=True)
    mask = torch.zeros(upair.numel(), **i64)
    mask.index_add_(0, inv, torch.bitwise_left_shift(torch.ones_like(key), key & 15))
    del key, inv
    prow = upair // n
    meta = (upair % n) | (mask << 24)
    cnt = torch.zeros_like(mask)
    for k in range(K):
        cnt += (mask >> k) & 1
    vstart = torch.cumsum(cnt, 0) - cnt
    rowcnt = torch.bincount(prow, minlength=n)
    return meta, vals, prow, rowcnt, vstart, cnt, total


def kgroup_layout(t: DeviceTransfer, warps_per_sm: int = None, split: int = None):
    """K-packed pairs with rows padded to 32 pairs, cut into pieces of <= split
    pairs, + cost-balanced warp ranges for sss_transfer_kgroup (built on the
    device)."""
    import os

    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_KGROUP_WPS", "24"))
    split = split or int(os.environ.get("SSS_KGROUP_SPLIT", "512"))
    split -= split % 32
    dev = t.rowptr.device
    n = t.n
    i64 = dict(dtype=torch.int64, device=dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 8
    meta, vals, prow, rowcnt, vstart, cnt, total = _kpacked_pairs(t)
    npairs = meta.numel()
    rowstart = torch.cumsum(rowcnt, 0) - rowcnt
    rowpad = (rowcnt + 31) // 32 * 32
    padstart = torch.cumsum(rowpad, 0) - rowpad
    npad = int(rowpad.sum().item())
    meta_p = torch.zeros(max(npad, 32), dtype=torch.int32, device=dev)
    meta = torch.where(meta >= (1 << 31), meta - (1 << 32), meta).to(torch.int32)
    meta_p[torch.arange(npairs, **i64) - rowstart[prow] + padstart[prow]] = meta
    # pieces
    npc = (rowcnt + split - 1) // split
    rep = torch.repeat_interleave(torch.arange(n, **i64), npc)
    j = torch.arange(rep.numel(), **i64) - (torch.cumsum(npc, 0) - npc)[rep]
    p0 = padstart[rep] + j * split
    pn = torch.minimum(torch.full_like(p0, split), rowpad[rep] - j * split)
    u0 = rowstart[rep] + j * split  # first real pair of the piece
    un = torch.clamp(torch.minimum(torch.full_like(u0, split), rowcnt[rep] - j * split), min=0)
    vend_all = torch.cat([vstart, torch.tensor([total], **i64)])
    v0 = vend_all[u0]
    nval = vend_all[u0 + un] - v0
    pieces = torch.stack([p0, pn, v0, rep], 1).to(torch.int32).contiguous()
    cost = pn * 2 + nval + 24  # meta + shuffles, values, per-piece overhead
    cum = torch.cat([torch.zeros(1, **i64), torch.cumsum(cost, 0)])
    targets = torch.arange(W + 1, dtype=torch.float64, device=dev) * (float(cum[-1]) / W)
    wbeg = torch.searchsorted(cum.to(torch.float64), targets, side="left")
    wbeg[-1] = p0.numel()
    stats = {"pairs": npairs, "padded_pairs": npad, "values": total, "pieces": int(p0.numel()),
             "max_row_pairs": int(rowcnt.max().item()),
             "bytes": npad * 4 + total * 4 + int(p0.numel()) * 16}
    return (meta_p, vals, pieces, wbeg.to(torch.int32).contiguous(), W, stats)


def block_column_order(side: int, levels: int, block: int = 2):
    """Column permutation for the flat8 gathers: tile-major w0 id -> an order
    where one 128-byte line of the packed x (4 columns x 32 B) holds the same
    tile-local coefficient of a block x block group of adjacent tiles, so the
    entries of a row that read one local coefficient of neighbouring source
    tiles share an L1 line. Returns (new_of_tm, tm_of_new) int64 arrays."""
    T = 1 << levels
    T2, tpr = T * T, side // T
    n = side * side
    tm = np.arange(n, dtype=np.int64)
    tile, local = tm // T2, tm % T2
    tr, tc = tile // tpr, tile % tpr
    bpr = max(tpr // block, 1)
    b = block if tpr >= block else 1
    bt = (tr // b) * bpr + (tc // b)
    q = (tr % b) * b + (tc % b)
    new = bt * (T2 * b * b) + local * (b * b) + q
    inv = np.empty_like(new)
    inv[new] = tm
    return new, inv


def flat_layout(t: DeviceTransfer, warps_per_sm: int = None, group: int = 4, interleave=None,
                col_order=None):
    """Head-flag bitmap + per-word segment prefix + segment (row, k) ids over
    csr9's padded operator copy, and equal word ranges per warp, for
    sss_transfer_flat."""
    import os

    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_FLAT_WPS", "16"))
    attr = "csr9" if group == 4 else f"csr9_pad{group}"
    if getattr(t, attr, None) is None:
        setattr(t, attr, csr9_layout(t, split=1 << 30, pad=group))
    pcols, pvals, pieces, _, _ = getattr(t, attr)
    dev = pcols.device
    if col_order is not None:
        # remap the columns and re-sort every segment by the new id (padding
        # entries, value 0, stay at their segment's end with column 0)
        new_of = torch.as_tensor(col_order, device=dev)
        pc0 = pieces.to(torch.int64) & 0xFFFFFFFF
        st, ln = pc0[:, 0], pc0[:, 1]
        seg = torch.repeat_interleave(torch.arange(st.numel(), device=dev), ln)
        pos = torch.arange(seg.numel(), device=dev, dtype=torch.int64)
        cl = new_of[pcols.to(torch.int64) & 0xFFFFFFFF]
        pad = pvals == 0
        key = (seg << 25) | torch.where(pad, torch.full_like(cl, (1 << 24) - 1 + 1), cl)
        order = torch.argsort(key, stable=True)
        pcols = torch.where(pad[order], torch.zeros_like(cl), cl[order]).to(torch.int32)
        pvals = pvals[order].contiguous()
        del seg, pos, cl, pad, key, order
    if interleave is None:
        interleave = group == 8 and os.environ.get("SSS_FLAT_INTERLEAVE", "1") == "1"
    if interleave:
        # lane-interleave every segment: with L = len / group lanes, entry
        # e * L + j goes to lane j, slot e, so gather instruction e reads L
        # consecutive (column-sorted, spatially clustered) entries instead of
        # entries `group` apart; each lane still holds one segment's entries
        pc0 = pieces.to(torch.int64) & 0xFFFFFFFF
        st, ln = pc0[:, 0], pc0[:, 1]
        seg = torch.repeat_interleave(torch.arange(st.numel(), device=dev), ln)
        q = torch.arange(int(ln.sum().item()), device=dev, dtype=torch.int64) - \
            torch.repeat_interleave(torch.cumsum(ln, 0) - ln, ln)
        L = (ln // group)[seg]
        src = st[seg] + q
        dst = st[seg] + (q % L) * group + q // L
        pc2, pv2 = pcols.clone(), pvals.clone()
        pc2[dst] = pcols[src]
        pv2[dst] = pvals[src]
        pcols, pvals = pc2, pv2
        del seg, q, L, src, dst
    i64 = dict(dtype=torch.int64, device=dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 8
    n_entries = pcols.numel()
    n4 = n_entries // group
    nw = (n4 + 31) // 32
    pc = pieces.to(torch.int64) & 0xFFFFFFFF
    s4 = pc[:, 0] // group
    heads = torch.zeros(nw, **i64).index_add_(0, s4 // 32, torch.bitwise_left_shift(
        torch.ones_like(s4), s4 % 32))
    heads = torch.where(heads >= (1 << 31), heads - (1 << 32), heads).to(torch.int32)
    cnt = torch.bincount(s4 // 32, minlength=nw)
    hpre = (torch.cumsum(cnt, 0) - cnt).to(torch.int32)
    rowk = pc[:, 2].to(torch.int32).contiguous()
    wbeg = (torch.arange(W + 1, **i64) * nw) // W
    stats = {"entries": n_entries, "words": nw, "segments": int(s4.numel()),
             "bytes": n_entries * 8 + nw * 8 + int(s4.numel()) * 4}
    return (pcols, pvals, n_entries, heads.contiguous(), hpre.contiguous(), rowk,
            wbeg.to(torch.int32).contiguous(), W, stats)


def flat8c_layout(t: DeviceTransfer, parts: int = None, ctas_per_sm: int = 2):
    """v22 column-partitioned flat8 stream (csrc/flat8c22.cu): entries sorted
    by (column partition, row, k, column), every (partition, row, k)
    sub-segment padded to a multiple of 8 entries, partition streams padded
    to whole 32-group words; 16-bit partition-local columns + f32 values;
    head bits / word prefixes / segment (row, k) ids as flat8; CTAs assigned
    to partitions in proportion to their words, the words of a partition
    split evenly over its CTAs' warps."""
    import os

    n, K = t.n, t.K
    parts = parts or int(os.environ.get("SSS_FLAT8C_PARTS", "16"))
    if n % parts or (n // parts) > 65536 or (n // parts) % 32:
        raise ValueError("flat8c: the column partition width must divide n, be a multiple of 32 "
                         "and fit 16 bits")
    cw = n // parts
    dev = t.rowptr.device
    rp = t.rowptr.to(torch.int64)
    nnz = int(rp[-1, -1])
    kk = torch.repeat_interleave(torch.arange(K, device=dev), rp[:, -1] - rp[:, 0])
    rows = torch.cat([torch.repeat_interleave(torch.arange(n, device=dev), torch.diff(rp[k]))
                      for k in range(K)])
    cols = t.cols[:nnz].to(torch.int64) & 0xFFFFFFFF
    part = cols // cw
    seg = (part * n + rows) * 16 + kk          # (partition, row, k) sub-segment key
    key = seg * n + cols
    del rows
    key, order = torch.sort(key)
    seg = key // n
    lcol = (key % n) % cw
    vals = t.vals[:nnz][order]
    del key, order, cols, kk, part
    useg, cnt = torch.unique_consecutive(seg, return_counts=True)
    plen = (cnt + 7) // 8 * 8                 # padded sub-segment lengths
    spart = useg // (16 * n)
    # partition streams padded to whole words (32 groups = 256 entries)
    pent = torch.zeros(parts, dtype=torch.int64, device=dev).index_add_(0, spart, plen)
    ppad = (pent + 255) // 256 * 256
    pbase = torch.zeros(parts + 1, dtype=torch.int64, device=dev)
    torch.cumsum(ppad, 0, out=pbase[1:])
    sstart_in_part = torch.cumsum(plen, 0) - plen
    # sub-segments are sorted partition-major: a partition's first one is at
    # the cumulative count of the partitions before it
    nseg_p = torch.bincount(spart, minlength=parts)
    first_idx = torch.cumsum(nseg_p, 0) - nseg_p
    first_of_part = torch.where(nseg_p > 0, sstart_in_part[torch.clamp(first_idx, max=max(
        0, sstart_in_part.numel() - 1))], torch.zeros_like(nseg_p))
    sstart = pbase[spart] + sstart_in_part - first_of_part[spart]
    total = int(pbase[-1])
    eseg = torch.repeat_interleave(torch.arange(useg.numel(), device=dev), cnt)
    pos = sstart[eseg] + (torch.arange(nnz, device=dev) - (torch.cumsum(cnt, 0) - cnt)[eseg])
    c16 = torch.zeros(total, dtype=torch.int16, device=dev)
    v32 = torch.zeros(total, dtype=torch.float32, device=dev)
    c16[pos] = lcol.to(torch.int32).to(torch.int16)
    v32[pos] = vals
    del eseg, pos, lcol, vals
    g0 = sstart // 8                            # first group of each sub-segment
    nwords = total // 256
    heads = torch.zeros(nwords, dtype=torch.int64, device=dev).index_add_(
        0, g0 // 32, torch.bitwise_left_shift(torch.ones_like(g0), g0 % 32))
    heads = torch.where(heads >= (1 << 31), heads - (1 << 32), heads).to(torch.int32)
    wc = torch.bincount(g0 // 32, minlength=nwords)
    hpre = (torch.cumsum(wc, 0) - wc).to(torch.int32)
    rowk = (useg % (16 * n)).to(torch.int32)    # row * 16 + k
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    G = nsm * ctas_per_sm
    pw = (ppad // 256).cpu()
    share = pw.double() / max(1, int(pw.sum())) * G
    cta_n = torch.clamp(share.floor().long(), min=1)
    while int(cta_n.sum()) < G:                 # largest remainders first
        cta_n[int(torch.argmax(share - cta_n.double()))] += 1
    while int(cta_n.sum()) > G:
        cta_n[int(torch.argmax(cta_n - share))] -= 1
    wpc = 512 // 32
    cta_part, wbeg = [], []
    pb = (pbase // 256).cpu()
    for p_ in range(parts):
        nw_ = int(cta_n[p_]) * wpc
        b0, b1 = int(pb[p_]), int(pb[p_ + 1])
        cta_part += [p_] * int(cta_n[p_])
        wbeg += [b0 + (b1 - b0) * j // nw_ for j in range(nw_)]
    wbeg.append(int(pb[-1]))
    stats = {"entries": total, "nnz": nnz, "parts": parts, "part_width": cw, "ctas": G,
             "bytes": total * 6 + nwords * 8 + int(useg.numel()) * 4}
    return (c16, v32, heads.contiguous(), hpre.contiguous(), rowk.contiguous(),
            torch.tensor(wbeg, dtype=torch.int32, device=dev),
            torch.tensor(cta_part, dtype=torch.int32, device=dev), G, parts, cw, stats)


def rbcsc_layout(t: DeviceTransfer, row_block: int = None):
    """v24 row-block column-major layout (csrc/rbcsc24.cu): per block of
    `row_block` tile-major rows, the entries of all K terms grouped by column
    (segments described by column | length << 16 and first entry), entries as
    (row in block | k << log2 row_block) u16 + f32 value; rowabs[k] = max over
    rows of sum |T_k[row, :]| (the fixed-point scale bound)."""
    import os

    n, K = t.n, t.K
    rb = row_block or int(os.environ.get("SSS_RBCSC_RB", "128"))
    if n > 65536 or K > 8 or n % rb:
        raise ValueError("rbcsc layout needs n <= 65536 (16-bit columns), K <= 8, rb | n")
    sh = rb.bit_length() - 1
    dev = t.rowptr.device
    rp = t.rowptr.to(torch.int64)
    nnz = int(rp[-1, -1])
    kk = torch.repeat_interleave(torch.arange(K, device=dev), rp[:, -1] - rp[:, 0])
    rows = torch.cat([torch.repeat_interleave(torch.arange(n, device=dev), torch.diff(rp[k]))
                      for k in range(K)])
    cols = t.cols[:nnz].to(torch.int64) & 0xFFFFFFFF
    vals = t.vals[:nnz]
    rowabs = torch.zeros(K * n, dtype=torch.float64, device=dev).index_add_(
        0, kk * n + rows, vals.abs().double()).view(K, n).amax(1).contiguous()
    key = ((rows // rb) * n + cols) * (rb * 8) + (kk * rb + rows % rb)
    key, order = torch.sort(key)
    rk16 = (((key % (rb * 8)) % rb) | (((key % (rb * 8)) // rb) << sh)).to(torch.int32)
    v32 = vals[order].contiguous()
    del order
    seg = key // (rb * 8)
    del key
    useg, cnt = torch.unique_consecutive(seg, return_counts=True)
    del seg
    first = torch.cumsum(cnt, 0) - cnt
    desc = torch.stack([((useg % n) | (cnt << 16)), first], 1)
    desc = torch.where(desc >= (1 << 31), desc - (1 << 32), desc).to(torch.int32).contiguous()
    blk = useg // n
    dcount = torch.bincount(blk, minlength=n // rb)
    dptr = torch.zeros(n // rb + 1, dtype=torch.int64, device=dev)
    torch.cumsum(dcount, 0, out=dptr[1:])
    stats = {"segments": int(useg.numel()), "entries": nnz, "row_block": rb,
             "bytes": nnz * 6 + int(useg.numel()) * 8}
    return (desc, dptr.to(torch.int32).contiguous(), rk16.to(torch.int16).contiguous(), v32,
            rowabs, rb, stats)


def kpairs_layout(t: DeviceTransfer, warps_per_sm: int = None):
    """v21 pair layout (csrc/kpairs21.cu): the K operators merged per (row,
    column) pair — header = column | term mask << 16, values pair-major with
    terms ascending — rows cut into chunks of <= 32 pairs, and whole-row warp
    ranges of about equal chunk count. Built on the device from the frame CSR."""
    import os

    n, K = t.n, t.K
    if n > 65536 or K > 8:
        raise ValueError("kpairs layout needs n <= 65536 and K <= 8")
    dev = t.rowptr.device
    rp = t.rowptr.to(torch.int64)
    nnz = int(rp[-1, -1])
    kk = torch.repeat_interleave(torch.arange(K, device=dev), rp[:, -1] - rp[:, 0])
    rows = torch.cat([torch.repeat_interleave(torch.arange(n, device=dev), torch.diff(rp[k]))
                      for k in range(K)])
    cols = t.cols[:nnz].to(torch.int64) & 0xFFFFFFFF
    key = (rows * n + cols) * 8 + kk
    del rows, cols
    key, order = torch.sort(key)
    vals = t.vals[:nnz][order].contiguous()
    del order
    pk = key >> 3                      # row * n + col
    kbit = torch.bitwise_left_shift(torch.ones_like(key), key & 7)
    del key
    first = torch.ones(nnz, dtype=torch.bool, device=dev)
    first[1:] = pk[1:] != pk[:-1]
    pid = torch.cumsum(first, 0) - 1
    npairs = int(pid[-1]) + 1 if nnz else 0
    mask = torch.zeros(npairs, dtype=torch.int64, device=dev).index_add_(0, pid, kbit)
    pstart = torch.nonzero(first).squeeze(1)          # value index of each pair's first term
    pkey = pk[pstart]
    del pk, kbit, first, pid
    prow = pkey // n
    hdr = ((pkey % n) | (mask << 16)).to(torch.int32)
    cnt = torch.bincount(prow, minlength=n)            # pairs per row
    pp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(cnt, 0, out=pp[1:])
    nch = torch.clamp((cnt + 31) // 32, min=1)         # every row >= 1 chunk
    cp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(nch, 0, out=cp[1:])
    C = int(cp[-1])
    crow = torch.repeat_interleave(torch.arange(n, device=dev), nch)
    ci = torch.arange(C, device=dev) - cp[crow]
    cfirst = pp[crow] + 32 * ci
    ccount = torch.clamp(pp[crow + 1] - cfirst, min=0, max=32)
    vstart = torch.cat([pstart, torch.tensor([nnz], device=dev)])
    cv = vstart[torch.clamp(cfirst, max=npairs)]
    chunks = torch.stack([crow, cfirst, ccount, cv], 1).to(torch.int32).contiguous()
    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_KPAIRS_WPS", "16"))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 8
    # whole-row warp ranges: warp w starts at the first row whose chunk prefix
    # reaches w * C / W
    target = (torch.arange(W + 1, device=dev, dtype=torch.int64) * C) // W
    rstart = torch.searchsorted(cp[:-1].contiguous(), target, right=False)
    rstart = torch.clamp(rstart, max=n)
    cbeg = cp[rstart]
    cbeg[-1] = C
    cbeg = torch.cummax(cbeg, 0).values
    stats = {"pairs": npairs, "chunks": C, "values": nnz,
             "bytes": npairs * 4 + nnz * 4 + C * 16, "kfill": nnz / max(1, npairs * K)}
    # per-row pair / value starts (the pair-group kernel's row table)
    t.kpairs_rows = (pp.to(torch.int32).contiguous(),
                     vstart[torch.clamp(pp, max=npairs)].to(torch.int32).contiguous())
    return chunks, hdr.contiguous(), vals, cbeg.to(torch.int32).contiguous(), W, stats


def pairgroup_layout(t: DeviceTransfer, warps_per_sm: int = None):
    """v23 (csrc/kgroup23.cu): the kpairs headers / values with per-row pair
    and value starts, and whole-row warp ranges of about equal pair counts."""
    import os

    if getattr(t, "kpairs", None) is None:
        t.kpairs = kpairs_layout(t)
    _, hdr, vals, _, _, st = t.kpairs
    pp, vp = t.kpairs_rows
    dev = pp.device
    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_PAIRGROUP_WPS", "48"))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 8
    n = t.n
    # cost of a row ~ its 8-pair steps + a fixed row overhead
    steps = (torch.diff(pp.to(torch.int64)) + 7) // 8 + 2
    cum = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(steps, 0, out=cum[1:])
    target = (torch.arange(W + 1, device=dev, dtype=torch.int64) * int(cum[-1])) // W
    rbeg = torch.clamp(torch.searchsorted(cum[:-1].contiguous(), target), max=n)
    rbeg[-1] = n
    rbeg = torch.cummax(rbeg, 0).values
    return pp, vp, hdr, vals, rbeg.to(torch.int32).contiguous(), W, dict(st, warps=W)


def regional_layout(t: DeviceTransfer, region_tiles: int = 1):
    """v19 layout: receiver regions (blocks of region_tiles x region_tiles
    2^L tiles, contiguous tile-major rows). Per region the sorted union of the
    columns its entries read (`ucols`, offsets `uoff`); the region's entries
    reference region-local slots instead of columns, in the flat8 stream
    (segments padded to 8, lane-interleaved) with every region padded to whole
    256-entry warp iterations (`rit` = iteration offsets per region).
    Returns a dict of device tensors + stats."""
    from types import SimpleNamespace

    dev = t.rowptr.device
    n, K, L = t.n, t.K, t.levels
    T2 = (1 << L) ** 2
    tpr = t.side >> L
    i64 = dict(dtype=torch.int64, device=dev)
    rp = t.rowptr.to(torch.int64)
    lens = (rp[:, 1:] - rp[:, :-1]).reshape(-1)
    base = int(rp[0, 0].item())
    total = int(lens.sum().item())
    kr = torch.arange(K * n, **i64)
    row = torch.repeat_interleave(kr % n, lens)
    col = t.cols[base:base + total].to(torch.int64) & 0xFFFFFFFF
    tile = row // T2
    rt = region_tiles
    if tpr % rt:
        raise ValueError("region_tiles must divide the tiles per row")
    region = (tile // tpr // rt) * (tpr // rt) + (tile % tpr) // rt
    # rows must be region-contiguous in tile-major order for a contiguous stream
    if rt != 1:
        raise ValueError("only single-tile regions keep rows contiguous in tile-major order")
    n_reg = n // T2
    key = region * n + col
    ukeys = torch.unique(key)
    ureg = ukeys // n
    ucols = (ukeys % n).to(torch.int32)
    ucnt = torch.bincount(ureg, minlength=n_reg)
    uoff = torch.cat([torch.zeros(1, **i64), torch.cumsum(ucnt, 0)])
    slot = torch.searchsorted(ukeys, key) - uoff[region]
    if int(ucnt.max().item()) >= 32768:
        raise ValueError("a region reads more than 32767 distinct columns")
    del key, ukeys, ureg, row, col, tile, region
    # the slot-valued operator (same rowptr / values), then the flat8 machinery
    cols_slot = t.cols.clone()
    cols_slot[base:base + total] = slot.to(torch.int32)
    del slot
    ts = SimpleNamespace(rowptr=t.rowptr, cols=cols_slot, vals=t.vals, n=n, K=K, levels=L,
                         side=t.side)
    # pad each region's last segment so regions span whole 32-group iterations
    lay = csr9_layout(ts, split=1 << 30, pad=8)
    pcols, pvals, pieces, _, _ = lay
    pc = pieces.to(torch.int64) & 0xFFFFFFFF
    st, ln, rk = pc[:, 0], pc[:, 1], pc[:, 2]
    preg = (rk >> 4) // T2
    reg_len = torch.zeros(n_reg, **i64).index_add_(0, preg, ln)
    reg_pad = (reg_len + 255) // 256 * 256 - reg_len
    last = torch.zeros(n_reg, **i64).scatter_reduce_(0, preg, torch.arange(ln.numel(), **i64), "amax")
    ln2 = ln.clone()
    ln2[last] += reg_pad
    st2 = torch.cumsum(ln2, 0) - ln2
    tot2 = int(ln2.sum().item())
    pc2 = torch.zeros(tot2, dtype=torch.int32, device=dev)
    pv2 = torch.zeros(tot2, dtype=torch.float32, device=dev)
    seg = torch.repeat_interleave(torch.arange(ln.numel(), device=dev), ln)
    q = torch.arange(int(ln.sum().item()), **i64) - torch.repeat_interleave(st, ln)
    pc2[st2[seg] + q] = pcols[st[seg] + q]
    pv2[st2[seg] + q] = pvals[st[seg] + q]
    del seg, q, pcols, pvals
    pieces2 = torch.stack([st2, ln2, rk, torch.zeros_like(rk)], 1).to(torch.int32).contiguous()
    ts.csr9_pad8 = (pc2, pv2, pieces2, None, 0)
    fl = flat_layout(ts, group=8, warps_per_sm=1)
    pcols_f, pvals_f, ne, heads, hpre, rowk, _, _, fst = fl
    reg_it = torch.cat([torch.zeros(1, **i64), torch.cumsum((reg_len + reg_pad) // 256, 0)])
    stats = {"regions": n_reg, "union_cols_mean": float(ucnt.float().mean()),
             "union_cols_max": int(ucnt.max()), "entries_padded": int(ne),
             "bytes": int(ne) * 8 + int(ucols.numel()) * 4}
    return {"pcols": pcols_f, "pvals": pvals_f, "n_entries": ne, "heads": heads, "hpre": hpre,
            "rowk": rowk, "ucols": ucols, "uoff": uoff.to(torch.int32).contiguous(),
            "rit": reg_it.to(torch.int32).contiguous(), "n_regions": n_reg,
            "umax": int(ucnt.max()), "stats": stats}


def k8_layout(t: DeviceTransfer, warps_per_sm: int = None, split: int = None):
    """v20 dense K-fused pairs: every (row, column) pair of the K operators
    once, its K <= 8 values in one 32-byte slot (0 for absent terms); rows
    padded to multiples of 32 pairs (column = N marks padding), cut into
    pieces of <= split pairs; cost-balanced per-warp piece ranges."""
    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_K8_WPS", "20"))
    split = split or int(os.environ.get("SSS_K8_SPLIT", "1024"))
    split -= split % 32
    if t.K > 8:
        raise ValueError("the dense K-fused layout needs K <= 8")
    dev = t.rowptr.device
    n, K = t.n, t.K
    i64 = dict(dtype=torch.int64, device=dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 8
    rp = t.rowptr.to(torch.int64)
    lens = (rp[:, 1:] - rp[:, :-1]).reshape(-1)
    base = int(rp[0, 0].item())
    total = int(lens.sum().item())
    kr = torch.arange(K * n, **i64)
    row_of = torch.repeat_interleave(kr % n, lens)
    k_of = torch.repeat_interleave(kr // n, lens)
    col = t.cols[base:base + total].to(torch.int64) & 0xFFFFFFFF
    upair, inv = torch.unique(row_of * n + col, return_inverse=True)
    del col
    prow = upair // n
    pcol = upair % n
    npairs = upair.numel()
    rowcnt = torch.bincount(prow, minlength=n)
    rowstart = torch.cumsum(rowcnt, 0) - rowcnt
    rowpad = (rowcnt + 31) // 32 * 32
    padstart = torch.cumsum(rowpad, 0) - rowpad
    npad = int(rowpad.sum().item())
    ppos = torch.arange(npairs, **i64) - rowstart[prow] + padstart[prow]
    cols_p = torch.full((max(npad, 32),), n, dtype=torch.int32, device=dev)
    cols_p[ppos] = pcol.to(torch.int32)
    vals_p = torch.zeros((max(npad, 32), 8), dtype=torch.float32, device=dev)
    vals_p[ppos[inv], k_of] = t.vals[base:base + total]
    del inv, k_of, row_of, upair, pcol
    npc = (rowpad + split - 1) // split
    rep = torch.repeat_interleave(torch.arange(n, **i64), npc)
    j = torch.arange(rep.numel(), **i64) - (torch.cumsum(npc, 0) - npc)[rep]
    p0 = padstart[rep] + j * split
    pn = torch.minimum(torch.full_like(p0, split), rowpad[rep] - j * split)
    pieces = torch.stack([p0, pn, rep, torch.zeros_like(rep)], 1).to(torch.int32).contiguous()
    cost = pn + 64
    cum = torch.cat([torch.zeros(1, **i64), torch.cumsum(cost, 0)])
    targets = torch.arange(W + 1, dtype=torch.float64, device=dev) * (float(cum[-1]) / W)
    wbeg = torch.searchsorted(cum.to(torch.float64), targets, side="left")
    wbeg[-1] = p0.numel()
    stats = {"pairs": npairs, "padded_pairs": npad, "pieces": int(p0.numel()),
             "bytes": npad * 36 + int(p0.numel()) * 16}
    return (cols_p, vals_p, pieces, wbeg.to(torch.int32).contiguous(), W, stats)


def kstep_layout(t: DeviceTransfer, warps_per_sm: int = None):
    """Mask-sorted K-fused warp steps for sss_transfer_kstep (built on the
    device): per row, (row, column) pairs sorted by (popcount, k-mask), cut
    into 32-pair steps; per step the columns and, for each k in the OR of the
    step's masks, 32 lane-ordered f32 values (0 where a pair lacks k)."""
    import os

    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_KSTEP_WPS", "20"))
    if t.K > 8:
        raise ValueError("kstep layout needs K <= 8")
    dev = t.rowptr.device
    n, K = t.n, t.K
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 4
    i64 = dict(dtype=torch.int64, device=dev)
    rp = t.rowptr.to(torch.int64)
    lens = (rp[:, 1:] - rp[:, :-1]).reshape(-1)
    base = int(rp[0, 0].item())
    total = int(lens.sum().item())
    kr = torch.arange(K * n, **i64)
    row_of = torch.repeat_interleave(kr % n, lens)
    k_of = torch.repeat_interleave(kr // n, lens)
    col = t.cols[base:base + total].to(torch.int64) & 0xFFFFFFFF
    ent_val = t.vals[base:base + total]
    # pairs in (row, col) order
    pkey = row_of * n + col
    upair, pinv = torch.unique(pkey, return_inverse=True)
    del pkey, col
    npairs = upair.numel()
    mask = torch.zeros(npairs, **i64)
    mask.index_add_(0, pinv, torch.bitwise_left_shift(torch.ones_like(k_of), k_of))
    prow = upair // n
    pcol = upair % n
    pc = torch.zeros_like(mask)
    for k in range(K):
        pc += (mask >> k) & 1
    # per row: sort by (popcount, mask), stable in column order
    skey = (prow << 12) | (pc << 8) | mask
    skey, order = torch.sort(skey, stable=True)
    del skey
    newpos = torch.empty_like(order)
    newpos[order] = torch.arange(npairs, **i64)
    prow_s, pcol_s, mask_s = prow[order], pcol[order], mask[order]
    del order
    rowcnt = torch.bincount(prow_s, minlength=n)
    rowstart = torch.cumsum(rowcnt, 0) - rowcnt
    pos = torch.arange(npairs, **i64) - rowstart[prow_s]
    nst = (rowcnt + 31) // 32
    ststart = torch.cumsum(nst, 0) - nst
    nsteps = int(nst.sum().item())
    step_of = ststart[prow_s] + pos // 32
    lane_of = pos % 32
    umask = torch.zeros(nsteps, **i64)
    for k in range(K):
        bit = ((mask_s >> k) & 1)
        has = torch.zeros(nsteps, **i64).scatter_reduce_(0, step_of, bit, "amax")
        umask |= has << k
    upc = torch.zeros_like(umask)
    for k in range(K):
        upc += (umask >> k) & 1
    val0 = (torch.cumsum(upc, 0) - upc) * 32
    nvals = int(upc.sum().item()) * 32
    # scatter every coefficient to its (step, rank of k, lane) slot
    p_new = newpos[pinv]
    st = step_of[p_new]
    below = umask[st] & (torch.bitwise_left_shift(torch.ones_like(k_of), k_of) - 1)
    rank = torch.zeros_like(below)
    for k in range(K):
        rank += (below >> k) & 1
    dest = val0[st] + rank * 32 + lane_of[p_new]
    vals_out = torch.zeros(max(nvals, 32), dtype=torch.float32, device=dev)
    vals_out[dest] = ent_val
    del p_new, st, below, rank, dest, pinv, k_of, row_of
    cols_out = pcol_s.to(torch.int32).contiguous()
    # step records
    srow = torch.repeat_interleave(torch.arange(n, **i64), nst)
    sidx = torch.arange(nsteps, **i64) - ststart[srow]
    pair0 = rowstart[srow] + sidx * 32
    count = torch.minimum(torch.full_like(pair0, 32), rowcnt[srow] - sidx * 32)
    row_end = (sidx == nst[srow] - 1).to(torch.int64)
    info = umask | (count << 8) | (row_end << 16)
    steps = torch.stack([pair0, val0, srow, info], 1).to(torch.int32).contiguous()
    cost = count + 32 * upc + 48  # columns + values + per-step overhead (in 4-byte units)
    cum = torch.cat([torch.zeros(1, **i64), torch.cumsum(cost, 0)])
    targets = torch.arange(W + 1, dtype=torch.float64, device=dev) * (float(cum[-1]) / W)
    wbeg = torch.searchsorted(cum.to(torch.float64), targets, side="left")
    wbeg[-1] = nsteps
    stats = {"pairs": npairs, "steps": nsteps, "values": nvals,
             "bytes": npairs * 4 + nvals * 4 + nsteps * 16}
    return (cols_out, vals_out, steps, wbeg.to(torch.int32).contiguous(), W, stats)


def kstream_layout(t: DeviceTransfer, warps_per_sm: int = None):
    """The kstep warp steps re-packed as contiguous per-step blobs for
    sss_transfer_kstream: [32 u32 columns | popc(mask) x 32 f32 values]."""
    import os

    warps_per_sm = warps_per_sm or int(os.environ.get("SSS_KSTREAM_WPS", "16"))
    cols, vals, steps, _, _, stats = kstep_layout(t, warps_per_sm=1)
    dev = cols.device
    i64 = dict(dtype=torch.int64, device=dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
    W = nsm * warps_per_sm
    W -= W % 8
    st = steps.to(torch.int64) & 0xFFFFFFFF
    pair0, val0, row, info = st[:, 0], st[:, 1], st[:, 2], st[:, 3]
    nsteps = st.shape[0]
    umask = info & 0xFF
    count = (info >> 8) & 0xFF
    upc = torch.zeros_like(umask)
    for k in range(8):
        upc += (umask >> k) & 1
    words = 32 * (1 + upc)  # 4-byte words per step blob
    off = torch.cumsum(words, 0) - words
    blob = torch.zeros(max(int(words.sum().item()), 4), dtype=torch.int32, device=dev)
    # columns (padded lanes stay 0)
    sid = torch.repeat_interleave(torch.arange(nsteps, **i64), count)
    lane = torch.arange(sid.numel(), **i64) - (torch.cumsum(count, 0) - count)[sid]
    blob[off[sid] + lane] = cols[pair0[sid] + lane]
    # values, already lane-ordered per k slot
    sid = torch.repeat_interleave(torch.arange(nsteps, **i64), 32 * upc)
    v = torch.arange(sid.numel(), **i64)
    blob[off[sid] + 32 + (v - val0[sid])] = vals[v].view(torch.int32)
    del sid, v, lane
    recs = torch.stack([off // 4, row, info, torch.zeros_like(off)], 1).to(torch.int32).contiguous()
    cost = words + 48
    cum = torch.cat([torch.zeros(1, **i64), torch.cumsum(cost, 0)])
    targets = torch.arange(W + 1, dtype=torch.float64, device=dev) * (float(cum[-1]) / W)
    wbeg = torch.searchsorted(cum.to(torch.float64), targets, side="left")
    wbeg[-1] = nsteps
    stats = dict(stats, bytes=int(blob.numel()) * 4 + nsteps * 16)
    return (blob, recs, wbeg.to(torch.int32).contiguous(), W, stats)


