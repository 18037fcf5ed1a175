"""PCIe bandwidth: H2D alone, D2H alone, and both at once (pinned host memory, separate streams)."""
import torch

n = 2 << 30   # 2 GiB per direction
h_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_src, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_dst.copy_(d_b, non_blocking=True)
    cur = torch.cuda.current_stream()
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return reps * n * (int(h2d) + int(d2h)) / ms / 1e6


run(True, True, 1)
print(f"H2D alone {run(True, False):.1f} GB/s, D2H alone {run(False, True):.1f} GB/s, "
      f"both {run(True, True):.1f} GB/s aggregate")
