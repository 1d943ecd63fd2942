"""Host <-> device copy bandwidth on this box (pinned, contiguous, 256 MB-2 GB),
H2D and D2H alone and concurrently -- the bound of bench.py's e2e leg."""
import torch

n = 1 << 30  # 1 GiB
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d.copy_(h, non_blocking=True)


def d2h():
    h2.copy_(d2, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for name, fn in (("H2D", h2d), ("D2H", d2h), ("H2D+D2H concurrent", both)):
    ms = t(fn)
    gb = n / 1e9 * (2 if name.startswith("H2D+") else 1)
    print(f"{name}: {ms:.2f} ms per GiB-each, {gb / (ms * 1e-3):.1f} GB/s total")
