"""Does a concurrent PCIe copy (17.3 MB, the cfg2 step's activations) slow kernels on another stream?
Compute = bf16 matmuls (~0.9 ms) on stream A; copies on streams B (H2D) / C (D2H)."""
import torch

n = (2048 + 64) * 4096
h_in = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
h_out = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
d_in = torch.empty(n, dtype=torch.bfloat16, device="cuda")
d_out = torch.randn(n, device="cuda").to(torch.bfloat16)
a = torch.randn(2112, 4096, device="cuda", dtype=torch.bfloat16)
w = torch.randn(14336 * 2, 4096, device="cuda", dtype=torch.bfloat16)
A, B, Cs = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def compute():
    for _ in range(2):
        (a @ w.t())


def run(h2d, d2h, reps=20):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if h2d:
            with torch.cuda.stream(B):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(Cs):
                h_out.copy_(d_out, non_blocking=True)
        with torch.cuda.stream(A):
            e[0].record(A)
            compute()
            e[1].record(A)
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]))
    ts.sort()
    return ts[len(ts) // 2]


for h2d, d2h in [(0, 0), (1, 0), (0, 1), (1, 1), (0, 0)]:
    print(f"overlap h2d={h2d} d2h={d2h}: compute {run(h2d, d2h):.3f} ms")
