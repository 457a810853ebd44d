"""Same-process A/B of library builds on forward attention through the C ABI (ctypes, RTLD_LOCAL):
per shape a CUDA graph of R launches per library, replayed alternately 9 times; min / median TFLOP/s.
python scripts/experiments/ab_attn_proc.py libA.so libB.so [libC.so ...]"""
import ctypes
import os
import statistics
import sys

import torch

paths = sys.argv[1:]
libs = [ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL) for p in paths]
for L in libs:
    L.cy_attention_fwd.restype = ctypes.c_int
    L.cy_attention_fwd.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_float, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
for causal, b, s in ((False, 2, 8192), (False, 8, 2048), (False, 16, 1024), (True, 1, 16384), (True, 4, 4096),
                     (True, 16, 1024)):
    h = 16
    Q, K, V = (torch.empty((b, h, s, 128), device="cuda", dtype=torch.float16).uniform_(-1, 1) for _ in range(3))
    O = torch.empty_like(Q)
    fl = 4.0 * b * h * s * s * 128 / (2 if causal else 1)
    reps = max(4, int(2e13 / fl))
    st = torch.cuda.Stream()
    graphs = []
    for L in libs:
        def launch():
            rc = L.cy_attention_fwd(0, b, h, s, s, 128, 128 ** -0.5, int(causal), Q.data_ptr(), K.data_ptr(),
                                    V.data_ptr(), O.data_ptr(), None, ctypes.c_void_p(st.cuda_stream))
            assert rc == 0, rc
        with torch.cuda.stream(st):
            for _ in range(3):
                launch()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                launch()
        graphs.append(g)
    times = [[] for _ in libs]
    for r in range(9):
        for j, g in enumerate(graphs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            times[j].append(e0.elapsed_time(e1) / reps)
    line = [f"{'c' if causal else 'n'}{b}x{s:<6d}"]
    for j, p in enumerate(paths):
        md = statistics.median(times[j])
        line.append(f"{os.path.basename(p)[10:22]:12s} {fl / md / 1e9:6.0f} (best {fl / min(times[j]) / 1e9:6.0f})")
    print(" | ".join(line), flush=True)
