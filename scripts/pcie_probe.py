"""PCIe probe: H2D of 108 MB (C1 bases + offsets per 1 M reads) alone, D2H of
24 MB (results) alone, and both at once on separate streams."""
import torch

x = torch.empty(108_000_000, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
r = torch.empty(24_000_000, dtype=torch.uint8, device="cuda")
rh = torch.empty(24_000_000, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d=True, d2h=True, chunks=16):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    ev[0].record(torch.cuda.current_stream())
    s1.wait_event(ev[0])
    s2.wait_event(ev[0])
    if h2d:
        with torch.cuda.stream(s1):
            n = x.numel() // chunks
            for i in range(chunks):
                y[i * n:(i + 1) * n].copy_(x[i * n:(i + 1) * n], non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            n = r.numel() // chunks
            for i in range(chunks):
                rh[i * n:(i + 1) * n].copy_(r[i * n:(i + 1) * n], non_blocking=True)
    ev[1].record(s1)
    ev[2].record(s2)
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]), ev[0].elapsed_time(ev[2])


for _ in range(3):
    run()
print("H2D alone  %.3f ms" % run(True, False)[0])
print("D2H alone  %.3f ms" % run(False, True)[1])
a, b = run()
print("both: H2D %.3f ms, D2H %.3f ms" % (a, b))
