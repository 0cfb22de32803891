"""compress_many / decompress_many -- the drop-in API over many fields.

The reference compresses many files by running ``codec.compress`` once per
file on a thread pool (``ebzip/cli.py:100-113``).  These two calls are that
loop for host-resident fields, pipelined on the B200:

    copy stream    H2D group g+1            H2D group g+2 ...
    compute        batched pipeline g       batched pipeline g+1 ...
    copy-out       (sizes of g known) D2H products / reconstructions of g

Fields of one geometry and dtype are processed ``group`` at a time through the
batched device pipelines (``ebz_compress_batch`` / ``ebz_decompress_batch_ptrs``:
one predict/quantize sweep launch per group).  Device memory is bounded by two
groups, whatever the number of fields: group g uses context slots, input
staging and output buffers of ring half g % 2, and waits (stream events) for
group g - 2 to have left them.  ``Context.trim()`` gives the workspaces back.  Results are the same objects
the single-field calls return, element for element identical; their arrays
(and ``code_bits``, a read-only ``memoryview``) live in pinned host memory so
the device writes them directly.  Mixed geometries fall back to the
single-field calls.  Errors are raised like the sequential loop would: the
first failing field's exception, after all in-flight work has finished.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from . import codec
from .core import CompressedStream, DataGrid, element_dtype, header_size

# context slots: the batches use two groups' worth from these bases (the
# one-shot calls use 1 << 20)
COMPRESS_SLOT = 2 << 20
DECOMPRESS_SLOT = 3 << 20


# Fields per pipelined group: about kGroupBytes of input per group.  Smaller
# groups shorten the pipeline's fill and drain (the first H2D and the last
# D2H run alone); measured on the cfg5 batch (64 x 67 MB, PCIe-bound at
# ~55 GB/s per direction): 16 fields/group 21.9 GB/s round trip, 8 -> 23.1,
# 4 -> 23.5, 2 -> 23.7.  Small fields keep up to 16 per group so each device
# batch still fills the GPU.
kGroupBytes = 256 << 20


def _auto_group(field_bytes: int) -> int:
    return max(2, min(16, kGroupBytes // max(1, int(field_bytes))))


def _pinned(nbytes: int):
    import torch
    return torch.empty(max(16, int(nbytes)), dtype=torch.uint8, pin_memory=True)


def _infos(nf: int):
    buf = _pinned(nf * ctypes.sizeof(nat.EbzInfo))
    return buf, (nat.EbzInfo * nf).from_address(buf.data_ptr())


def _trusted_stream(width, dims, layers, m, eb, lengths, nbits, bits, unpred):
    """CompressedStream around device-produced, already consistent parts."""
    st = object.__new__(CompressedStream)
    st.element_width = width
    st.dims = tuple(int(v) for v in dims)
    st.layers = int(layers)
    st.interval_exponent = int(m)
    st.eb_effective = float(eb)
    st.code_lengths = lengths
    st.code_bit_length = int(nbits)
    st.code_bits = bits
    st.unpredictable_values = unpred
    return st


def compress_many(grids, config, *, group: int | None = None, device: int | None = None):
    """``[codec.compress(g, config) for g in grids]``, pipelined."""
    grids = list(grids)
    if not grids:
        return []
    g0 = grids[0]
    if config.truncate_unpredictable or any(g.dims != g0.dims or g.values.dtype != g0.values.dtype
                                            for g in grids):
        # (the opt-in truncated coding runs through the single-field calls)
        return [codec.compress(g, config, device=device) for g in grids]
    import torch
    ctx = nat.context(device)
    dev = torch.device("cuda", ctx.device)
    nf, n, width = len(grids), g0.n_values, g0.element_width
    ew, m, ndim = width // 8, config.interval_exponent, g0.ndim
    group = group or _auto_group(n * ew)
    dims = nat.dims_array(g0.dims)
    ha, av, hr, rv = codec._bound_args(config)
    hsz = header_size(ndim)
    vals = [np.ascontiguousarray(g.values) for g in grids]
    group = min(group, nf)
    # input staging: ring of two groups
    d_in = torch.empty((2, group, n), dtype=torch.float32 if width == 32 else torch.float64,
                       device=dev)
    info_buf, infos = _infos(nf)
    groups = [list(range(i, min(i + group, nf))) for i in range(0, nf, group)]
    s_copy, s_comp, s_out = (torch.cuda.Stream(dev) for _ in range(3))
    ev_in = [torch.cuda.Event() for _ in groups]
    ev_c = [torch.cuda.Event() for _ in groups]
    ev_f = [torch.cuda.Event() for _ in groups]
    arenas = [None] * len(groups)
    lib, h = ctx.lib, ctx.handle

    def slot(gi, i):  # field i of group gi
        return COMPRESS_SLOT + (gi % 2) * group + (i - groups[gi][0])

    def fetch(gi):
        ev_c[gi].synchronize()
        idx = groups[gi]
        sizes = []
        for i in idx:
            inf = infos[i]
            bad = inf.status & (nat.ST_NONFINITE_IN | nat.ST_EB_NONPOSITIVE | nat.ST_EMPTY_HIST |
                                nat.ST_DEPTH_GT_64)
            nb = 0 if bad else (int(inf.bit_length) + 7) // 8
            nu = 0 if bad else int(inf.n_unpred) * ew
            sizes.append((hsz + (1 << m), nb, nu))
        offs, tot = [], 0
        for a, b, c in sizes:
            offs.append((tot, tot + ((a + 15) & ~15), tot + ((a + 15) & ~15) + ((b + 15) & ~15)))
            tot += ((a + 15) & ~15) + ((b + 15) & ~15) + ((c + 15) & ~15)
        arena = _pinned(tot)
        arenas[gi] = (arena, offs, sizes)
        base = arena.data_ptr()
        s_out.wait_event(ev_c[gi])
        for i, (o_h, o_b, o_u), (a, b, c) in zip(idx, offs, sizes):
            if b == 0 and infos[i].status:
                continue
            ctx.check(lib.ebz_compress_fetch_async(
                h, slot(gi, i), ctypes.byref(infos[i]), ctypes.c_void_p(base + o_h),
                ctypes.c_void_p(base + o_b), ctypes.c_void_p(base + o_u), s_out.cuda_stream),
                "ebz_compress_fetch_async")
        ev_f[gi].record(s_out)

    with ctx.lock:
        for gi, idx in enumerate(groups):
            stage = d_in[gi % 2]
            if gi >= 2:  # ring half gi % 2: group gi - 2 has read its inputs ...
                s_copy.wait_event(ev_c[gi - 2])
            for k, i in enumerate(idx):
                ctx.check(lib.ebz_copy_async(h, ctypes.c_void_p(stage[k].data_ptr()),
                                             ctypes.c_void_p(vals[i].ctypes.data), n * ew,
                                             s_copy.cuda_stream), "ebz_copy_async")
            ev_in[gi].record(s_copy)
            s_comp.wait_event(ev_in[gi])
            if gi >= 2:  # ... and its products have left the slots
                s_comp.wait_event(ev_f[gi - 2])
            ptrs = (ctypes.c_void_p * len(idx))(*[stage[k].data_ptr() for k in range(len(idx))])
            ctx.check(lib.ebz_compress_batch(h, slot(gi, idx[0]), len(idx), ptrs, width,
                                             ndim, dims, config.layers, m, ha, av, hr, rv,
                                             s_comp.cuda_stream), "ebz_compress_batch")
            for i in idx:
                ctx.check(lib.ebz_slot_info_async(h, slot(gi, i), 0,
                                                  ctypes.c_void_p(ctypes.addressof(infos[i])),
                                                  s_comp.cuda_stream), "ebz_slot_info_async")
            ev_c[gi].record(s_comp)
            if gi >= 1:
                fetch(gi - 1)
        fetch(len(groups) - 1)
        s_out.synchronize()

    outs = []
    dtype = element_dtype(width)
    for gi, idx in enumerate(groups):
        arena, offs, sizes = arenas[gi]
        a_np = arena.numpy()
        for i, (o_h, o_b, o_u), (a, b, c) in zip(idx, offs, sizes):
            inf = infos[i]
            codec._raise_compress_status(inf)
            head = a_np[o_h:o_h + a]
            bits = memoryview(a_np[o_b:o_b + b]).toreadonly()
            unpred = a_np[o_u:o_u + c].view(dtype)
            unpred.flags.writeable = False
            st = _trusted_stream(width, g0.dims, config.layers, m, inf.eb,
                                 head[hsz:hsz + (1 << m)], inf.bit_length, bits, unpred)
            outs.append(codec._outcome_of(st, n, config, inf))
    return outs


def decompress_many(streams, *, group: int | None = None, device: int | None = None):
    """``[codec.decompress(s) for s in streams]``, pipelined."""
    streams = list(streams)
    if not streams:
        return []
    s0 = streams[0]
    key = (s0.element_width, tuple(s0.dims), s0.layers, s0.interval_exponent)
    if any((s.element_width, tuple(s.dims), s.layers, s.interval_exponent) != key
           for s in streams):
        return [codec.decompress(s, device=device) for s in streams]
    for s in streams:
        codec._validate_table(s.code_lengths)
    import torch
    ctx = nat.context(device)
    dev = torch.device("cuda", ctx.device)
    nf, n, width = len(streams), s0.n_points, s0.element_width
    ew, m, ndim = width // 8, s0.interval_exponent, len(s0.dims)
    group = group or _auto_group(n * ew)
    dims = nat.dims_array(s0.dims)
    dtype = element_dtype(width)
    group = min(group, nf)
    groups = [list(range(i, min(i + group, nf))) for i in range(0, nf, group)]
    # device inputs, per group: lengths | bits (+64 B slack) | verbatim, at
    # offsets within the group's arena; two arenas (ring halves) sized for
    # the largest group of each parity
    nbytes = [len(s.code_bits) for s in streams]
    ks = [s.n_unpredictable for s in streams]
    off_b, off_u = [0] * nf, [0] * nf
    tb_max, tu_max = [256, 256], [256, 256]
    for gi, idx in enumerate(groups):
        tb = tu = 0
        for i in idx:
            off_b[i] = tb
            tb += (nbytes[i] + 64 + 255) & ~255
            off_u[i] = tu
            tu += (max(ks[i], 1) * ew + 255) & ~255
        tb_max[gi % 2] = max(tb_max[gi % 2], tb)
        tu_max[gi % 2] = max(tu_max[gi % 2], tu)
    d_len = torch.empty((2, group, 1 << m), dtype=torch.uint8, device=dev)
    d_bits = [torch.zeros(tb_max[r], dtype=torch.uint8, device=dev) for r in range(2)]
    d_unp = [torch.empty(tu_max[r], dtype=torch.uint8, device=dev) for r in range(2)]
    d_rec = torch.empty((2, group, n), dtype=torch.float32 if width == 32 else torch.float64,
                        device=dev)
    h_rec = _pinned(nf * n * ew)
    info_buf, infos = _infos(nf)
    s_copy, s_comp, s_out = (torch.cuda.Stream(dev) for _ in range(3))
    ev_in = [torch.cuda.Event() for _ in groups]
    ev_c = [torch.cuda.Event() for _ in groups]
    ev_o = [torch.cuda.Event() for _ in groups]
    lib, h = ctx.lib, ctx.handle
    lens = [np.ascontiguousarray(s.code_lengths, np.uint8) for s in streams]
    bits_h = [np.frombuffer(s.code_bits, np.uint8) if nb else None
              for s, nb in zip(streams, nbytes)]
    unp_h = [np.ascontiguousarray(s.unpredictable_values, dtype) for s in streams]
    cp = lambda dst, src, nb: ctx.check(  # noqa: E731
        lib.ebz_copy_async(h, ctypes.c_void_p(dst), ctypes.c_void_p(src), nb,
                           s_copy.cuda_stream), "ebz_copy_async")
    with ctx.lock:
        for gi, idx in enumerate(groups):
            r = gi % 2
            dl, db, du, dr = d_len[r], d_bits[r], d_unp[r], d_rec[r]
            if gi >= 2:  # ring half r: group gi - 2 has read its inputs ...
                s_copy.wait_event(ev_c[gi - 2])
            for k, i in enumerate(idx):
                cp(dl[k].data_ptr(), lens[i].ctypes.data, 1 << m)
                if nbytes[i]:
                    cp(db.data_ptr() + off_b[i], bits_h[i].ctypes.data, nbytes[i])
                if ks[i]:
                    cp(du.data_ptr() + off_u[i], unp_h[i].ctypes.data, ks[i] * ew)
            ev_in[gi].record(s_copy)
            s_comp.wait_event(ev_in[gi])
            if gi >= 2:  # ... and its reconstructions have left for the host
                s_comp.wait_event(ev_o[gi - 2])
            g = len(idx)
            arr = lambda vals, t: (t * g)(*vals)  # noqa: E731
            ctx.check(lib.ebz_decompress_batch_ptrs(
                h, DECOMPRESS_SLOT + r * group, g, width, ndim, dims, s0.layers, m,
                arr([float(streams[i].eb_effective) for i in idx], ctypes.c_double),
                arr([ks[i] for i in idx], ctypes.c_uint64),
                arr([dl[k].data_ptr() for k in range(g)], ctypes.c_void_p),
                arr([db.data_ptr() + off_b[i] for i in idx], ctypes.c_void_p),
                arr([nbytes[i] for i in idx], ctypes.c_uint64),
                arr([du.data_ptr() + off_u[i] for i in idx], ctypes.c_void_p),
                arr([dr[k].data_ptr() for k in range(g)], ctypes.c_void_p),
                s_comp.cuda_stream), "ebz_decompress_batch_ptrs")
            for k, i in enumerate(idx):
                ctx.check(lib.ebz_slot_info_async(h, DECOMPRESS_SLOT + r * group + k, 1,
                                                  ctypes.c_void_p(ctypes.addressof(infos[i])),
                                                  s_comp.cuda_stream), "ebz_slot_info_async")
            ev_c[gi].record(s_comp)
            s_out.wait_event(ev_c[gi])
            ctx.check(lib.ebz_copy_async(
                h, ctypes.c_void_p(h_rec.data_ptr() + idx[0] * n * ew),
                ctypes.c_void_p(dr[0].data_ptr()), g * n * ew, s_out.cuda_stream),
                "ebz_copy_async")
            ev_o[gi].record(s_out)
        s_out.synchronize()
    rec = h_rec.numpy()[: nf * n * ew].view(dtype).reshape(nf, n)
    out = []
    for i, s in enumerate(streams):
        codec._raise_decompress_status(infos[i], s, nbytes[i])
        out.append(codec._trusted_grid(s.dims, rec[i]))
    return out
