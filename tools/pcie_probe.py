"""PCIe copy bandwidth of this box (pinned host <-> HBM, 17.3 MB = the cfg2 step's activations),
each direction alone and both at once on two streams: the bound on bench.py's e2e leg."""
import torch

n = (2048 + 64) * 4096
h_in = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
h_out = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
d_in = torch.empty(n, dtype=torch.bfloat16, device="cuda")
d_out = torch.randn(n, device="cuda").to(torch.bfloat16)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


by = n * 2
for name, fn in [("h2d", lambda: d_in.copy_(h_in, non_blocking=True)),
                 ("d2h", lambda: h_out.copy_(d_out, non_blocking=True)), ("both", both)]:
    t = timed(fn)
    print(f"pcie {name}: {by / 1e6:.1f} MB per direction in {t * 1e3:.3f} ms -> {by / t / 1e9:.1f} GB/s per direction")
