"""Host-buffer codec pipeline: encode / decode packet-major stripes that live in
(pinned) host memory, overlapping PCIe copies in both directions with the
GPU kernels.

The stripes are cut into chunks; chunk c runs on stream c % nstreams as
  H2D(source) -> encode -> D2H(encoded)            (encode_host)
  H2D(received) -> decode -> D2H(decoded)          (decode_host)
so the H2D copy engine, the D2H copy engine and the SMs work on different
chunks at the same time. Plans are built once per call on the first stream
and every decode stream waits for them. This is the public entry point for
data that is not already resident in HBM (the reference CLI's use case:
files in, shards out); all arithmetic still runs in libfntrs_b200.so.
"""
from __future__ import annotations

import numpy as np

from .codec import Codec, Plans, default_escape_capacity


class HostPipeline:
    def __init__(self, codec: Codec, k: int, n: int, L: int, max_chunk_stripes: int, nstreams: int = 3,
                 systematic: bool = False):
        import torch
        self.torch, self.codec, self.systematic = torch, codec, systematic
        self.k, self.n, self.L = k, n, L
        self.chunk = max(1, max_chunk_stripes)
        dev = torch.device(f"cuda:{codec.device}")
        self.dev = dev
        self.streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
        c = self.chunk
        # per-stream device buffers (reused across chunks on the same stream)
        self.d_in = [torch.empty((c, k, L), dtype=torch.int16, device=dev) for _ in self.streams]
        self.d_enc = [torch.empty((c, n, L), dtype=torch.int16, device=dev) for _ in self.streams]
        self.d_dec = [torch.empty((c, k, L), dtype=torch.int16, device=dev) for _ in self.streams]
        cap_e = default_escape_capacity(c * n * L)
        self.cap_e = cap_e
        self.d_esc = [torch.empty(cap_e, dtype=torch.int64, device=dev) for _ in self.streams]
        self.d_cnt = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in self.streams]

    def _chunks(self, S):
        return [(a, min(S, a + self.chunk)) for a in range(0, S, self.chunk)]

    def encode_host(self, src_h, enc_h, esc_h, counts_h):
        """src_h [S,k,L] int16 pinned -> enc_h [S,n,L] int16 pinned. Chunk c's escape list
        (indices into its own [stripes][n][L] block) lands in esc_h[c], its count in counts_h[c]."""
        torch = self.torch
        S = src_h.shape[0]
        for c, (a, b) in enumerate(self._chunks(S)):
            i = c % len(self.streams)
            st = self.streams[i]
            with torch.cuda.stream(st):
                d_in, d_enc = self.d_in[i][: b - a], self.d_enc[i][: b - a]
                d_in.copy_(src_h[a:b], non_blocking=True)
                self.codec.encode(self.k, self.n, d_in, out=d_enc, esc_out=self.d_esc[i], esc_cap=self.cap_e,
                                  count=self.d_cnt[i], stream=st, systematic=self.systematic)
                enc_h[a:b].copy_(d_enc, non_blocking=True)
                esc_h[c].copy_(self.d_esc[i], non_blocking=True)
                counts_h[c:c + 1].copy_(self.d_cnt[i], non_blocking=True)

    def decode_host(self, plans: Plans, stripe_pattern_dev, rx_h, rx_esc_dev, dec_h, esc_h, counts_h,
                    esc_ranges=None):
        """rx_h [S,k,L] pinned -> dec_h [S,k,L] pinned. rx_esc_dev: sorted escape indices into rx
        (device, or None); esc_ranges[c] = (lo, hi) slice of it for chunk c, re-based per chunk."""
        torch = self.torch
        S = rx_h.shape[0]
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.dev))  # plans were built on the current stream
        for c, (a, b) in enumerate(self._chunks(S)):
            i = c % len(self.streams)
            st = self.streams[i]
            st.wait_event(ready)
            with torch.cuda.stream(st):
                d_rx, d_dec = self.d_in[i][: b - a], self.d_dec[i][: b - a]
                d_rx.copy_(rx_h[a:b], non_blocking=True)
                esc = None
                if rx_esc_dev is not None and esc_ranges is not None:
                    lo, hi = esc_ranges[c]
                    if hi > lo:
                        esc = rx_esc_dev[lo:hi] - a * self.k * self.L
                self.codec.decode(plans, stripe_pattern_dev[a:b], d_rx, esc, out=d_dec, esc_out=self.d_esc[i],
                                  esc_cap=self.cap_e, count=self.d_cnt[i], stream=st, systematic=self.systematic)
                dec_h[a:b].copy_(d_dec, non_blocking=True)
                esc_h[c].copy_(self.d_esc[i], non_blocking=True)
                counts_h[c:c + 1].copy_(self.d_cnt[i], non_blocking=True)

    def code_host(self, src_h, enc_h, enc_esc_h, enc_counts_h, plans: Plans, stripe_pattern_dev, rx_h, rx_esc_dev,
                  dec_h, dec_esc_h, dec_counts_h, esc_ranges=None):
        """encode_host and decode_host with their chunks interleaved on the
        streams (encode chunk c, then decode chunk c): the encode's heavy D2H
        (2n bytes per codeword) overlaps the decode's H2D, so both copy engines
        stay busy. The received packets must not depend on this call's encode
        (they are the erasure channel's output of an earlier one)."""
        torch = self.torch
        S = src_h.shape[0]
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.dev))
        ns = len(self.streams)
        for c, (a, b) in enumerate(self._chunks(S)):
            for phase in (0, 1):
                i = (2 * c + phase) % ns
                st = self.streams[i]
                if phase:
                    st.wait_event(ready)
                with torch.cuda.stream(st):
                    if phase == 0:
                        d_in, d_enc = self.d_in[i][: b - a], self.d_enc[i][: b - a]
                        d_in.copy_(src_h[a:b], non_blocking=True)
                        self.codec.encode(self.k, self.n, d_in, out=d_enc, esc_out=self.d_esc[i], esc_cap=self.cap_e,
                                          count=self.d_cnt[i], stream=st, systematic=self.systematic)
                        enc_h[a:b].copy_(d_enc, non_blocking=True)
                        enc_esc_h[c].copy_(self.d_esc[i], non_blocking=True)
                        enc_counts_h[c:c + 1].copy_(self.d_cnt[i], non_blocking=True)
                    else:
                        d_rx, d_dec = self.d_in[i][: b - a], self.d_dec[i][: b - a]
                        d_rx.copy_(rx_h[a:b], non_blocking=True)
                        esc = None
                        if rx_esc_dev is not None and esc_ranges is not None:
                            lo, hi = esc_ranges[c]
                            if hi > lo:
                                esc = rx_esc_dev[lo:hi] - a * self.k * self.L
                        self.codec.decode(plans, stripe_pattern_dev[a:b], d_rx, esc, out=d_dec, esc_out=self.d_esc[i],
                                          esc_cap=self.cap_e, count=self.d_cnt[i], stream=st,
                                          systematic=self.systematic)
                        dec_h[a:b].copy_(d_dec, non_blocking=True)
                        dec_esc_h[c].copy_(self.d_esc[i], non_blocking=True)
                        dec_counts_h[c:c + 1].copy_(self.d_cnt[i], non_blocking=True)

    def join(self):
        """Make the current stream wait for all pipeline streams."""
        cur = self.torch.cuda.current_stream(self.dev)
        for st in self.streams:
            ev = self.torch.cuda.Event()
            ev.record(st)
            cur.wait_event(ev)


def escape_ranges(rx_esc_host: np.ndarray, S: int, chunk: int, k: int, L: int):
    """(lo, hi) index ranges of a sorted escape list per chunk of `chunk` stripes."""
    if rx_esc_host is None or len(rx_esc_host) == 0:
        return [(0, 0)] * ((S + chunk - 1) // chunk)
    bounds = np.arange(0, S + chunk, chunk, dtype=np.int64)
    bounds[-1] = min(bounds[-1], S)
    cuts = np.searchsorted(rx_esc_host, np.minimum(bounds, S) * k * L)
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(len(cuts) - 1)]
