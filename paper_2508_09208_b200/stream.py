"""Host-to-host serving path: pinned host batches -> HBM -> MoE layer -> host.

Copy and compute streams form a depth-2 pipeline so the PCIe upload of
batch i+1, the layer forward of batch i and the download of batch i-1
overlap (PCIe is full duplex). Each 100 MB copy is split into 4 chunks over
2 streams per direction: one cudaMemcpyAsync reached 27.7 GB/s H2D, chunked
54.9 GB/s, ~47 GB/s per direction with both directions busy
(scripts/pcie_probe.py on a B200 box). Each batch is a complete layer
forward — routing, capacity
and outputs are exactly those of `MoELayer.forward` on that batch; only the
copies move off the critical path. This is the end-to-end call bench.py
times for its `e2e` figure.
"""

from __future__ import annotations

import torch


class HostPipeline:
    def __init__(self, layer, tokens: int, d_model: int, depth: int = 2, device=None,
                 chunks: int = 4, copy_streams: int = 2, graphs: bool = False):
        self.layer = layer
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.depth = depth
        self.x = [torch.empty((tokens, d_model), dtype=torch.bfloat16, device=self.dev)
                  for _ in range(depth)]
        self.y = [torch.empty_like(self.x[0]) for _ in range(depth)]
        self.chunks = max(1, chunks)
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_comp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.s_in_x = [self.s_in] + [torch.cuda.Stream(self.dev) for _ in range(copy_streams - 1)]
        self.s_out_x = [self.s_out] + [torch.cuda.Stream(self.dev) for _ in range(copy_streams - 1)]
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_comp = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self._used = [False] * depth
        # graphs: one captured forward per device buffer pair (MoELayer.capture)
        self.graphs = [layer.capture(self.x[k], self.y[k]) for k in range(depth)] if graphs else None

    def run(self, xs_host, ys_host, start_event=None, end_event=None):
        """Process pinned host batches xs_host[i] -> ys_host[i] (same shapes).
        Optional timing events are recorded on the upload stream before the
        first copy and on the download stream after the last copy."""
        if start_event is not None:
            start_event.record(self.s_in)
            for st in self.s_in_x[1:]:
                st.wait_event(start_event)
        for i, (xh, yh) in enumerate(zip(xs_host, ys_host)):
            k = i % self.depth
            self._copy(self.s_in_x, self.ev_comp[k] if self._used[k] else None,
                       self.x[k], xh)  # x[k] free once batch i-depth consumed it
            self.ev_in[k].record(self.s_in)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(self.ev_in[k])
                if self._used[k]:
                    self.s_comp.wait_event(self.ev_out[k])  # y[k] downloaded
                if self.graphs is not None:
                    self.graphs[k].replay()
                else:
                    self.layer.forward(self.x[k], out=self.y[k])
                self.ev_comp[k].record(self.s_comp)
            self._copy(self.s_out_x, self.ev_comp[k], yh, self.y[k])
            self.ev_out[k].record(self.s_out)
            self._used[k] = True
        if end_event is not None:
            for k in range(self.depth):
                if self._used[k]:
                    self.s_out.wait_event(self.ev_out[k])
            end_event.record(self.s_out)

    def _copy(self, streams, after, dst, src):
        """dst.copy_(src) as `chunks` row blocks spread over `streams`; the
        first stream ends up waiting for all of them."""
        rows = dst.shape[0]
        step = (rows + self.chunks - 1) // self.chunks
        head = streams[0]
        evs = []
        for c in range(self.chunks):
            lo, hi = c * step, min(rows, (c + 1) * step)
            if lo >= hi:
                break
            st = streams[c % len(streams)]
            with torch.cuda.stream(st):
                if after is not None:
                    st.wait_event(after)
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
                if st is not head:
                    ev = torch.cuda.Event()
                    ev.record(st)
                    evs.append(ev)
        for ev in evs:
            head.wait_event(ev)

    def synchronize(self):
        for s in (*self.s_in_x, self.s_comp, *self.s_out_x):
            s.synchronize()
