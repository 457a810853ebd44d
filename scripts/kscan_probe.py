"""Device time per GEMM launch (CUDA-graph replay, no host in the loop) vs K at fixed M=N, per config."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_07004_b200 as cy


def graph_time(fn, reps=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    mn = int(sys.argv[1]) if len(sys.argv) > 1 else 1536
    cfgs = [int(c) for c in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "3"])]
    for k in (64, 256, 512, 1024, 1536, 3072):
        a = torch.empty((mn, k), device="cuda", dtype=torch.float16).uniform_(-1, 1)
        b = torch.empty((k, mn), device="cuda", dtype=torch.float16).uniform_(-1, 1)
        d = torch.empty((mn, mn), device="cuda", dtype=torch.float16)
        line = [f"M=N={mn} K={k:5d}:"]
        for c in cfgs:
            cy.force_config(c)
            line.append(f"c{c} {graph_time(lambda: cy.gemm(a, b, out=d)):7.2f}")
        cy.force_config(-1)
        line.append(f"torch {graph_time(lambda: torch.matmul(a, b, out=d)):7.2f} us")
        print(" ".join(line), flush=True)


if __name__ == "__main__":
    main()
