"""Device-resident batch driver: many fields, many streams, no host syncs.

The drop-in API (``codec.compress`` / ``codec.decompress``) takes host
arrays; this module drives the same C-ABI pipelines on inputs that already
live in HBM (torch CUDA tensors used as plain buffers), which is how the
throughput of the path itself is measured and how a GPU-resident caller
would batch independent fields (the reference's file-level parallelism,
``ebzip/cli.py:100-113``, mapped onto CUDA streams).

Slots: field i compresses into context slot i (its products stay resident
for the decompress leg); decompression uses slots ``nfields + (i % S)``.
"""

from __future__ import annotations

import ctypes

from . import _native as nat


class DeviceBatch:
    def __init__(self, nstreams: int = 8, device: int | None = None):
        import torch
        self.torch = torch
        self.ctx = nat.context(device)
        self.device = torch.device("cuda", self.ctx.device)
        self.streams = [torch.cuda.Stream(device=self.device) for _ in range(nstreams)]

    # -- enqueue helpers ----------------------------------------------------
    def _stream(self, i):
        return self.streams[i % len(self.streams)]

    def compress_async(self, i, field, dims, config):
        """Enqueue compress of one device field (float32/float64 tensor) into slot i."""
        b = config.bound
        width = 32 if field.dtype == self.torch.float32 else 64
        rc = self.ctx.lib.ebz_compress_async(
            self.ctx.handle, i, field.data_ptr(), width, len(dims), nat.dims_array(dims),
            config.layers, config.interval_exponent,
            1 if b.absolute is not None else 0, float(b.absolute or 0.0),
            1 if b.relative is not None else 0, float(b.relative or 0.0),
            self._stream(i).cuda_stream)
        self.ctx.check(rc, "ebz_compress_async")

    def decompress_async(self, i, nfields, out):
        """Enqueue decompress of slot i's products into device tensor ``out``."""
        rc = self.ctx.lib.ebz_decompress_async(
            self.ctx.handle, nfields + (i % len(self.streams)), i, out.data_ptr(),
            self._stream(i).cuda_stream)
        self.ctx.check(rc, "ebz_decompress_async")

    def fork(self):
        cur = self.torch.cuda.current_stream(self.device)
        for s in self.streams:
            s.wait_stream(cur)

    def join(self):
        cur = self.torch.cuda.current_stream(self.device)
        for s in self.streams:
            cur.wait_stream(s)

    def compress_batch(self, fields, dims, config, slot0=0):
        """One batched compress of equally shaped device fields into slots
        slot0.. (single sweep launch for all fields; per-field stages on the
        library's worker streams), enqueued on the current stream."""
        b = config.bound
        width = 32 if fields[0].dtype == self.torch.float32 else 64
        ptrs = (ctypes.c_void_p * len(fields))(*[f.data_ptr() for f in fields])
        rc = self.ctx.lib.ebz_compress_batch(
            self.ctx.handle, slot0, len(fields), ptrs, width, len(dims), nat.dims_array(dims),
            config.layers, config.interval_exponent,
            1 if b.absolute is not None else 0, float(b.absolute or 0.0),
            1 if b.relative is not None else 0, float(b.relative or 0.0),
            self.torch.cuda.current_stream(self.device).cuda_stream)
        self.ctx.check(rc, "ebz_compress_batch")

    def decompress_batch(self, outs, src_slot0=0, slot0=None):
        """One batched decompress of slots src_slot0.. into device tensors."""
        if slot0 is None:
            slot0 = src_slot0 + len(outs)
        ptrs = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        rc = self.ctx.lib.ebz_decompress_batch(
            self.ctx.handle, slot0, src_slot0, len(outs), ptrs,
            self.torch.cuda.current_stream(self.device).cuda_stream)
        self.ctx.check(rc, "ebz_decompress_batch")

    # -- one timed pass -------------------------------------------------------
    def roundtrip(self, fields, dims, config, outs, batched=True, split=1):
        """Compress every field, then decompress every field (device resident).
        Returns CUDA events (start, compressed, decompressed) recorded on the
        current stream.  batched=False drives one pipeline per field on
        ``nstreams`` streams instead of the batched entry points.

        split > 1: the fields form ``split`` contiguous groups, each a batched
        compress then decompress on its own stream, so one group's stages
        fill the SMs another group's wavefront tail or serial stages leave
        idle.  The middle event then only marks the enqueue order (the legs
        overlap); the round trip is e0 -> e2."""
        torch = self.torch
        cur = torch.cuda.current_stream(self.device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        if batched and split > 1:
            nf = len(fields)
            per = (nf + split - 1) // split
            e0.record(cur)
            self.fork()
            with self.ctx.lock:
                for g, i0 in enumerate(range(0, nf, per)):
                    st = self.streams[g % len(self.streams)]
                    with torch.cuda.stream(st):
                        self.compress_batch(fields[i0:i0 + per], dims, config, slot0=i0)
                        self.decompress_batch(outs[i0:i0 + per], src_slot0=i0,
                                              slot0=nf + i0)
            e1.record(cur)
            self.join()
            e2.record(cur)
            return e0, e1, e2
        if batched:
            e0.record(cur)
            with self.ctx.lock:
                self.compress_batch(fields, dims, config)
                e1.record(cur)
                self.decompress_batch(outs)
            e2.record(cur)
            return e0, e1, e2
        e0.record(cur)
        self.fork()
        with self.ctx.lock:
            for i, f in enumerate(fields):
                self.compress_async(i, f, dims, config)
            self.join()
            e1.record(cur)
            self.fork()
            for i in range(len(fields)):
                self.decompress_async(i, len(fields), outs[i])
        self.join()
        e2.record(cur)
        return e0, e1, e2

    def info(self, slot) -> nat.EbzInfo:
        h = nat.EbzInfo()
        self.ctx.check(self.ctx.lib.ebz_slot_info(self.ctx.handle, slot, ctypes.byref(h), None),
                       "ebz_slot_info")
        return h

    def decode_info(self, slot) -> nat.EbzInfo:
        """Decompress record of a slot (status, verbatim values consumed)."""
        h = nat.EbzInfo()
        self.ctx.check(self.ctx.lib.ebz_slot_decode_info(self.ctx.handle, slot, ctypes.byref(h),
                                                         None), "ebz_slot_decode_info")
        return h

    def container(self, slot) -> bytes:
        """Serialized container of a compressed slot (D2H of its products)."""
        import numpy as np
        from .core import header_size
        h = self.info(slot)
        head_buf = np.empty(header_size(4) + (1 << 16), np.uint8)
        bits = np.empty((int(h.bit_length) + 7) // 8, np.uint8)
        # element width from the header written on the device
        self.ctx.check(self.ctx.lib.ebz_compress_fetch(self.ctx.handle, slot, nat.ptr(head_buf),
                                                       nat.ptr(bits), None, None),
                       "ebz_compress_fetch")
        ndim = int(head_buf[6])
        m = int(head_buf[7])
        width = 64 if head_buf[5] else 32
        head = head_buf[: header_size(ndim) + (1 << m)]
        unpred = np.empty(int(h.n_unpred), np.float64 if width == 64 else np.float32)
        self.ctx.check(self.ctx.lib.ebz_compress_fetch(self.ctx.handle, slot, None, None,
                                                       nat.ptr(unpred) if unpred.size else None,
                                                       None), "ebz_compress_fetch")
        return head.tobytes() + bits.tobytes() + unpred.tobytes()
