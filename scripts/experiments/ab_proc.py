"""Same-process A/B of two library builds through the C ABI (ctypes, RTLD_LOCAL): for each shape a
CUDA graph of R launches per library, replayed alternately 7 times; prints min / median us per launch.
python scripts/experiments/ab_proc.py libA.so libB.so SHAPES   (SHAPES e.g. b64,b64c,2048,8192;
b64c = batched with beta = 1)"""
import ctypes
import os
import statistics
import sys

import torch

libs = [ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL) for p in sys.argv[1:3]]
for L in libs:
    L.cy_gemm_batched.restype = ctypes.c_int
    L.cy_gemm_batched.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_float, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_int64,
                                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
u = lambda *s: torch.empty(s, device="cuda", dtype=torch.float16).uniform_(-1, 1)  # noqa
for sh in sys.argv[3].split(","):
    if sh.startswith("b"):
        beta = 1.0 if sh.endswith("c") else 0.0
        Lb = int(sh[1:].rstrip("c"))
        m = n = k = 1024
        sets = [(u(Lb, m, k), u(Lb, k, n), u(Lb, m, n)) for _ in range(4)]
        D = u(Lb, m, n)
        reps = 20
    else:
        Lb, beta = 1, 0.0
        m = n = k = int(sh)
        sets = [(u(m, k), u(k, n), u(m, n)) for _ in range(2)]
        D = u(m, n)
        reps = max(5, min(50, int(2e12 / (2.0 * m * n * k) * 20)))
    fl = 2.0 * Lb * m * n * k
    s = torch.cuda.Stream()
    graphs = []
    for L in libs:
        def launch(i):
            a, b_, c = sets[i % len(sets)]
            rc = L.cy_gemm_batched(0, m, n, k, Lb, 1.0, a.data_ptr(), k, m * k, b_.data_ptr(), n, k * n, beta,
                                   c.data_ptr(), n, m * n, D.data_ptr(), n, m * n, ctypes.c_void_p(s.cuda_stream))
            assert rc == 0, rc
        with torch.cuda.stream(s):
            for i in range(3):
                launch(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                launch(i)
        graphs.append(g)
    times = [[], []]
    for r in range(7):
        for j, g in enumerate(graphs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            times[j].append(e0.elapsed_time(e1) / reps * 1e3)
    line = [f"{sh:6s}"]
    for j in range(2):
        mn, md = min(times[j]), statistics.median(times[j])
        line.append(f"{os.path.basename(sys.argv[1 + j])[:16]:16s} min {mn:8.2f} med {md:8.2f} us ({fl / md / 1e6:6.0f} TF)")
    print(" | ".join(line), flush=True)
