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

``HostPipeline`` is the same schedule for any entry point of the library: ``fn(ins, outs, stream)``
enqueues the call on ``stream`` reading the device copies of the step's inputs and writing the
device outputs that are then downloaded.
"""
from __future__ import annotations

import torch

from . import gemm


class HostPipeline:
    """Three-stream overlap of upload / call / download for host-resident inputs and outputs.

    ``in_specs`` / ``out_specs``: lists of (shape, dtype) of the device buffers; ``fn(ins, outs,
    stream)`` enqueues one call of the library on ``stream``; ``alloc(shape, dtype)`` makes a device
    buffer (default: contiguous).  ``depth`` buffer sets rotate, ordered by CUDA events only."""

    def __init__(self, in_specs, out_specs, fn, device="cuda", depth: int = 2, alloc=None):
        self.device = torch.device(device)
        self.fn = fn
        self.depth = depth
        with torch.cuda.device(self.device):
            mk = alloc or (lambda shape, dtype: torch.empty(shape, dtype=dtype, device=self.device))
            self.h2d = torch.cuda.Stream(self.device)
            self.comp = torch.cuda.Stream(self.device)
            self.d2h = torch.cuda.Stream(self.device)
            self.ins = [[mk(sh, dt) for sh, dt in in_specs] for _ in range(depth)]
            self.outs = [[mk(sh, dt) for sh, dt in out_specs] for _ in range(depth)]
            # per slot: inputs uploaded, call done (inputs free, outputs ready), outputs downloaded
            self.ev_in = [torch.cuda.Event() for _ in range(depth)]
            self.ev_comp = [torch.cuda.Event() for _ in range(depth)]
            self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.i = 0
        self.used = [False] * depth

    def submit(self, host_ins, host_outs) -> None:
        """Queue one call: upload ``host_ins``, run ``fn``, download into ``host_outs`` (pinned host
        tensors overlap; the call returns immediately)."""
        s = self.i % self.depth
        self.i += 1
        if self.used[s]:
            self.h2d.wait_event(self.ev_comp[s])   # the call that read this slot's inputs is done
        with torch.cuda.stream(self.h2d):
            for dev, host in zip(self.ins[s], host_ins):
                dev.copy_(host, non_blocking=True)
            self.ev_in[s].record(self.h2d)
        self.comp.wait_event(self.ev_in[s])
        if self.used[s]:
            self.comp.wait_event(self.ev_out[s])   # this slot's previous outputs have been downloaded
        self.fn(self.ins[s], self.outs[s], self.comp)
        self.ev_comp[s].record(self.comp)
        self.d2h.wait_event(self.ev_comp[s])
        with torch.cuda.stream(self.d2h):
            for host, dev in zip(host_outs, self.outs[s]):
                host.copy_(dev, non_blocking=True)
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


class HostGemmPipeline(HostPipeline):
    """``HostPipeline`` for ``D = alpha * A @ B`` (device rows padded to 16-byte multiples)."""

    def __init__(self, m: int, n: int, k: int, dtype=torch.float16, device="cuda", depth: int = 2,
                 alpha: float = 1.0):
        self.alpha = alpha

        def alloc(shape, dt):
            rows, cols = shape
            return torch.empty((rows, (cols + 7) // 8 * 8), dtype=dt, device=device)[:, :cols]

        super().__init__([((m, k), dtype), ((k, n), dtype)], [((m, n), dtype)],
                         lambda ins, outs, st: gemm(ins[0], ins[1], alpha=self.alpha, out=outs[0], stream=st),
                         device=device, depth=depth, alloc=alloc)

    def submit(self, A_host: torch.Tensor, B_host: torch.Tensor, D_host: torch.Tensor) -> None:
        """Queue D_host <- alpha * A_host @ B_host (host tensors should be pinned for overlap)."""
        super().submit((A_host, B_host), (D_host,))
