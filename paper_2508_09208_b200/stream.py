"""Host-to-host serving path: pinned host batches -> HBM -> MoE layer -> host.

Three CUDA streams form a depth-2 pipeline so the PCIe upload of batch i+1,
the layer forward of batch i and the download of batch i-1 overlap (PCIe is
full duplex). Each batch is a complete layer forward — routing, capacity
and outputs are exactly those of `MoELayer.forward` on that batch; only the
copies move off the critical path. This is the end-to-end call bench.py
times for its `e2e` figure.
"""

from __future__ import annotations

import torch


class HostPipeline:
    def __init__(self, layer, tokens: int, d_model: int, depth: int = 2, device=None):
        self.layer = layer
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.depth = depth
        self.x = [torch.empty((tokens, d_model), dtype=torch.bfloat16, device=self.dev)
                  for _ in range(depth)]
        self.y = [torch.empty_like(self.x[0]) for _ in range(depth)]
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_comp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_comp = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self._used = [False] * depth

    def run(self, xs_host, ys_host, start_event=None, end_event=None):
        """Process pinned host batches xs_host[i] -> ys_host[i] (same shapes).
        Optional timing events are recorded on the upload stream before the
        first copy and on the download stream after the last copy."""
        if start_event is not None:
            start_event.record(self.s_in)
        for i, (xh, yh) in enumerate(zip(xs_host, ys_host)):
            k = i % self.depth
            with torch.cuda.stream(self.s_in):
                if self._used[k]:
                    self.s_in.wait_event(self.ev_comp[k])  # x[k] consumed by batch i-depth
                self.x[k].copy_(xh, non_blocking=True)
                self.ev_in[k].record(self.s_in)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(self.ev_in[k])
                if self._used[k]:
                    self.s_comp.wait_event(self.ev_out[k])  # y[k] downloaded
                self.layer.forward(self.x[k], out=self.y[k])
                self.ev_comp[k].record(self.s_comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_comp[k])
                yh.copy_(self.y[k], non_blocking=True)
                self.ev_out[k].record(self.s_out)
            self._used[k] = True
        if end_event is not None:
            for k in range(self.depth):
                if self._used[k]:
                    self.s_out.wait_event(self.ev_out[k])
            end_event.record(self.s_out)

    def synchronize(self):
        for s in (self.s_in, self.s_comp, self.s_out):
            s.synchronize()
