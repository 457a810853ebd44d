"""A/B of the library's environment tuning knobs (read once at load, so one process per setting).
    python scripts/experiments/knob_ab.py REPS WORKLOADS 'CY_GROUP_M=4' 'CY_GROUP_M=6 CY_SERP=0' 'CY_KNOBS_LIB=other.so' ...
WORKLOADS: comma list of batched, batched1 (beta=1), batched16 (L2-resident 16 x 1024^3), gN (N^3, short), gNs
(N^3, 3000 launches), rr65536.
Settings run interleaved, REPS rounds, on build/exp/libcypress_knobs.so
(scripts/build_experiment.py knobs CY_TUNING_KNOBS=1); prints us/launch and TFLOP/s per (setting, workload)."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
    import torch

    import paper_2504_07004_b200 as cy
    from paper_2504_07004_b200 import _lib

    # the product library reads no knobs: use the CY_TUNING_KNOBS experiment build
    _lib.use_library(os.environ.get("CY_KNOBS_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..",
                                                                 "build", "exp", "libcypress_knobs.so")))

    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.float16

    def rnd(*s):
        return torch.empty(s, device="cuda", dtype=h).uniform_(-1, 1, generator=g)

    def timeit(fn, iters, flops):
        for i in range(5):
            fn(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(iters):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / iters * 1e3
        return us, flops / us / 1e6

    for w in sys.argv[2].split(","):
        if w in ("batched", "batched1", "batched16"):
            L = 16 if w == "batched16" else 64  # batched16: one L2-resident set of 16 x 1024^3
            ns = 1 if w == "batched16" else 4
            sets = [(rnd(L, 1024, 1024), rnd(L, 1024, 1024), rnd(L, 1024, 1024)) for _ in range(ns)]
            D = torch.empty((L, 1024, 1024), device="cuda", dtype=h)
            beta = 1.0 if w == "batched1" else 0.0
            r = timeit(lambda i: cy.gemm_batched(sets[i % ns][0], sets[i % ns][1], sets[i % ns][2], 1.0, beta, out=D),
                       200, 2.0 * L * 1024 ** 3)
        elif w.startswith("g"):
            # gN: short (burst clock); gNs: 3000 launches (~2 s, power-capped clock)
            sus = w.endswith("s")
            n = int(w[1:].rstrip("s"))
            sets = [(rnd(n, n), rnd(n, n)) for _ in range(2)]
            D = torch.empty((n, n), device="cuda", dtype=h)
            r = timeit(lambda i: cy.gemm(sets[i % 2][0], sets[i % 2][1], out=D),
                       3000 if sus else max(20, int(4e13 / n ** 3)), 2.0 * n ** 3)
        elif w == "rr65536":
            A, B = rnd(65536, 8192), rnd(8192, 8192)
            D = torch.empty((65536, 8192), device="cuda", dtype=h)
            y = torch.empty(65536, device="cuda", dtype=torch.float32)
            r = timeit(lambda i: cy.gemm_rowreduce(A, B, out=D, y=y), 20, 2.0 * 65536 * 8192 ** 2)
        else:
            raise SystemExit(f"unknown workload {w}")
        print(f"{w} {r[0]:.2f} {r[1]:.1f}", flush=True)
    sys.exit(0)

reps, works, settings = int(sys.argv[1]), sys.argv[2], sys.argv[3:]
res = {}
for rep in range(reps):
    for s in settings:
        env = dict(os.environ)
        for kv in s.split():
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, __file__, "--child", works], env=env, capture_output=True, text=True)
        if out.returncode:
            print(f"[{s}] failed: {out.stderr[-800:]}", flush=True)
            continue
        for line in out.stdout.split("\n"):
            if line.strip():
                w, us, tf = line.split()
                res.setdefault((s, w), []).append((float(us), float(tf)))
                print(f"rep{rep} [{s:28s}] {w:9s} {float(us):9.2f} us {float(tf):8.1f} TF/s", flush=True)
print("---- best of reps")
for (s, w), v in sorted(res.items(), key=lambda kv: (kv[0][1], kv[0][0])):
    b = min(v)
    print(f"{w:9s} [{s:28s}] best {b[0]:9.2f} us {b[1]:8.1f} TF/s   median {sorted(x[0] for x in v)[len(v) // 2]:9.2f} us")
