"""Host-buffer forward with the PCIe transfers overlapped (the end-to-end call a
serving process makes when activations live in host memory).

The batch is split into chunks of `chunk` sequences; chunk c runs

    h2d stream:     x (and q, k unless the weights project them) pinned host
                    -> device slot c % depth
    compute stream: the MCA layer stack on that slot (libmca_b200 kernels)
    d2h stream:     y -> pinned host

so the copies of chunk c+1, the forward of chunk c and the read-back of chunk
c-1 proceed together. Chunk c passes b_offset + c * chunk, so its Philox
streams are those of the unsplit call and the output is bitwise the one
`mca_forward` gives on the whole batch. torch supplies the
streams, events and pinned/device memory only.
"""
from __future__ import annotations

import torch

from .api import AttentionWeights, McaConfig, mca_forward


class HostPipeline:
    def __init__(self, layers: list[AttentionWeights], n: int, chunk: int, dtype: torch.dtype,
                 device: torch.device | str = "cuda", depth: int = 4):
        if not layers:
            raise ValueError("need at least one layer")
        self.layers = layers
        self.n, self.chunk, self.depth = int(n), int(chunk), int(depth)
        self.device = torch.device(device)
        HD = layers[0].heads * layers[0].d_h
        d_in = layers[0].d_in
        if len(layers) > 1 and d_in != HD:
            raise ValueError("stacked layers feed y back as x: need d_in == heads * d_h")
        mk = lambda c: torch.empty((self.chunk, self.n, c), dtype=dtype, device=self.device)  # noqa: E731
        self.slots = [dict(q=mk(HD), k=mk(HD), x=mk(d_in), y=mk(HD), y2=mk(HD)) for _ in range(self.depth)]
        self.project = all(w.has_projections for w in layers)
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_comp = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)
        ev = lambda: [torch.cuda.Event() for _ in range(self.depth)]  # noqa: E731
        self.loaded, self.computed, self.freed = ev(), ev(), ev()
        self.used = [False] * self.depth

    def forward(self, hq: torch.Tensor | None, hk: torch.Tensor | None, hx: torch.Tensor, hy: torch.Tensor,
                cfg: McaConfig | None = None, seed: int = 0, b_offset: int = 0, sync: bool = True) -> None:
        """hq, hk: [B, n, H*64] (None: the weights carry W_q / W_k and only x is
        transferred), hx: [B, n, d_in] pinned host tensors; writes hy
        [B, n, H*64] (pinned host). Asynchronous: returns once the work is
        enqueued. sync=True: the caller's current stream waits for hy
        (stream-ordered, like one mca_forward). sync=False: it does not, so
        back-to-back calls pipeline across calls too (the next call's H2D and
        forward overlap this call's D2H; slots are reused only after their
        read-back); `wait()` joins the current stream to every read-back."""
        B = hx.shape[0]
        if hq is None and not self.project:
            raise ValueError("q / k omitted but the layers carry no W_q / W_k")
        if hx.shape[1] != self.n or B % self.chunk:
            raise ValueError(f"batch [{B}, {hx.shape[1]}] does not split into chunks of {self.chunk} x {self.n}")
        cur = torch.cuda.current_stream(self.device)
        for st in (self.s_h2d, self.s_comp, self.s_d2h):
            st.wait_stream(cur)   # device-side inputs / weights the caller enqueued before this call
        for c in range(B // self.chunk):
            i = c % self.depth
            sl = self.slots[i]
            rows = slice(c * self.chunk, (c + 1) * self.chunk)
            with torch.cuda.stream(self.s_h2d):
                if self.used[i]:
                    self.s_h2d.wait_event(self.freed[i])          # the slot's previous read-back finished
                if hq is not None:
                    sl["q"].copy_(hq[rows], non_blocking=True)
                    sl["k"].copy_(hk[rows], non_blocking=True)
                sl["x"].copy_(hx[rows], non_blocking=True)
                self.loaded[i].record(self.s_h2d)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(self.loaded[i])
                xin, bufs = sl["x"], (sl["y"], sl["y2"])
                for l, w in enumerate(self.layers):
                    out = bufs[l & 1]
                    qq, kk = (sl["q"], sl["k"]) if hq is not None else (None, None)
                    mca_forward(w, qq, kk, xin, cfg, seed, b_offset=b_offset + c * self.chunk, layer=l,
                                y=out, stream=self.s_comp)
                    xin = out
                self.computed[i].record(self.s_comp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(self.computed[i])
                hy[rows].copy_(xin, non_blocking=True)
                self.freed[i].record(self.s_d2h)
            self.used[i] = True
        if sync:
            cur.wait_stream(self.s_d2h)

    def wait(self) -> None:
        """The caller's current stream waits for every read-back enqueued so far."""
        torch.cuda.current_stream(self.device).wait_stream(self.s_d2h)
