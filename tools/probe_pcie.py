"""Dev probe: pinned host <-> device copy rates (the floor of bench.py's e2e number).
Copies 256 MiB (the cfg2 step's inputs / outputs) H2D alone, D2H alone and both at once on
two streams, CUDA-event timed; prints GB/s per direction."""
import torch

NB = 256 << 20
dev = torch.device("cuda:0")
h_in = torch.empty(NB, dtype=torch.uint8).pin_memory()
h_out = torch.empty(NB, dtype=torch.uint8).pin_memory()
d_in = torch.empty(NB, dtype=torch.uint8, device=dev)
d_out = torch.empty(NB, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream(dev)
    e0.record(cur)
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    for _ in range(reps):
        fn()
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("duplex", both)):
    ms = timed(fn)
    print("%-6s %.3f ms per 256 MiB each way -> %.1f GB/s per direction" % (name, ms, NB / ms / 1e6), flush=True)
