"""Host-streaming GEMM pipeline: overlap host->device copies, the sm_100a kernel and device->host
copies of consecutive GEMMs on three CUDA streams.

For inputs that live in (pinned) host memory the end-to-end cost of one GEMM is
H2D(A, B) + kernel + D2H(D); issued back to back they serialise.  ``HostGemmPipeline`` keeps
``depth`` device buffer sets and runs step i's kernel while step i+1's operands are uploaded and
step i-1's result is downloaded, so the steady-state time per step is the slowest of the three
(usually PCIe H2D).  Ordering is by CUDA events only (no host synchronisation inside ``submit``).

    pipe = HostGemmPipeline(m, n, k, dtype=torch.float16, device="cuda")
    for A_h, B_h, D_h in work:          # pinned host tensors
        pipe.submit(A_h, B_h, D_h)      # returns immediately
    pipe.synchronize()                  # every D_h is filled
"""
from __future__ import annotations

import torch

from . import gemm


class HostGemmPipeline:
    def __init__(self, m: int, n: int, k: int, dtype=torch.float16, device="cuda", depth: int = 2,
                 alpha: float = 1.0):
        self.device = torch.device(device)
        self.alpha = alpha
        self.depth = depth
        ldn = (n + 7) // 8 * 8
        ldk = (k + 7) // 8 * 8
        with torch.cuda.device(self.device):
            self.h2d = torch.cuda.Stream(self.device)
            self.comp = torch.cuda.Stream(self.device)
            self.d2h = torch.cuda.Stream(self.device)
            self.A = [torch.empty((m, ldk), dtype=dtype, device=self.device)[:, :k] for _ in range(depth)]
            self.B = [torch.empty((k, ldn), dtype=dtype, device=self.device)[:, :n] for _ in range(depth)]
            self.D = [torch.empty((m, ldn), dtype=dtype, device=self.device)[:, :n] for _ in range(depth)]
            # per slot: inputs uploaded, kernel done (inputs free, D ready), result downloaded (D free)
            self.ev_in = [torch.cuda.Event() for _ in range(depth)]
            self.ev_comp = [torch.cuda.Event() for _ in range(depth)]
            self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.i = 0
        self.used = [False] * depth

    def submit(self, A_host: torch.Tensor, B_host: torch.Tensor, D_host: torch.Tensor) -> None:
        """Queue D_host <- alpha * A_host @ B_host (host tensors should be pinned for overlap)."""
        s = self.i % self.depth
        self.i += 1
        if self.used[s]:
            self.h2d.wait_event(self.ev_comp[s])   # the kernel that read this slot's inputs is done
        with torch.cuda.stream(self.h2d):
            self.A[s].copy_(A_host, non_blocking=True)
            self.B[s].copy_(B_host, non_blocking=True)
            self.ev_in[s].record(self.h2d)
        self.comp.wait_event(self.ev_in[s])
        if self.used[s]:
            self.comp.wait_event(self.ev_out[s])   # this slot's previous result has been downloaded
        gemm(self.A[s], self.B[s], alpha=self.alpha, out=self.D[s], stream=self.comp)
        self.ev_comp[s].record(self.comp)
        self.d2h.wait_event(self.ev_comp[s])
        with torch.cuda.stream(self.d2h):
            D_host.copy_(self.D[s], non_blocking=True)
            self.ev_out[s].record(self.d2h)
        self.used[s] = True

    def wait_for(self, stream) -> None:
        """Make the pipeline's streams start after the work queued so far on ``stream``."""
        ev = torch.cuda.Event()
        ev.record(stream)
        for st in (self.h2d, self.comp, self.d2h):
            st.wait_event(ev)

    def join(self, stream) -> None:
        """Make ``stream`` wait for everything submitted so far (e.g. to time with events on it)."""
        stream.wait_stream(self.h2d)
        stream.wait_stream(self.comp)
        stream.wait_stream(self.d2h)

    def synchronize(self) -> None:
        for st in (self.h2d, self.comp, self.d2h):
            st.synchronize()
