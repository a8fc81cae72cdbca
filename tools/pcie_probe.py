"""PCIe copy rates on this box: pinned H2D alone, D2H alone, and both at once
on two streams (full duplex?), 1 GiB per copy, CUDA events."""
import torch

N = 1 << 27  # doubles = 1 GiB
h_in = torch.empty(N, dtype=torch.float64, pin_memory=True).fill_(1.0)
h_out = torch.empty(N, dtype=torch.float64, pin_memory=True)
d_in = torch.empty(N, dtype=torch.float64, device="cuda")
d_out = torch.empty(N, dtype=torch.float64, device="cuda").fill_(2.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fns, reps=4):
    torch.cuda.synchronize()
    ev = []
    for s, f in fns:
        with torch.cuda.stream(s):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                f()
            e1.record()
            ev.append((e0, e1))
    torch.cuda.synchronize()
    return [reps * N * 8 / (a.elapsed_time(b) * 1e-3) / 1e9 for a, b in ev]


h2d = lambda: d_in.copy_(h_in, non_blocking=True)
d2h = lambda: h_out.copy_(d_out, non_blocking=True)
timed([(s1, h2d)], 1)
print("H2D alone  %.1f GB/s" % timed([(s1, h2d)])[0])
print("D2H alone  %.1f GB/s" % timed([(s1, d2h)])[0])
a, b = timed([(s1, h2d), (s2, d2h)])
print("concurrent H2D %.1f GB/s  D2H %.1f GB/s" % (a, b))

# two H2D copies at once (two copy engines?) and chunk-size sweep of one H2D stream
h_in2 = torch.empty(N, dtype=torch.float64, pin_memory=True).fill_(3.0)
d_in2 = torch.empty(N, dtype=torch.float64, device="cuda")
h2d2 = lambda: d_in2.copy_(h_in2, non_blocking=True)
a, b = timed([(s1, h2d), (s2, h2d2)])
print("two H2D at once %.1f + %.1f GB/s" % (a, b))
for mb in (8, 32, 128, 512):
    k = mb * (1 << 20) // 8
    parts = [(d_in[i:i + k], h_in[i:i + k]) for i in range(0, N, k)]

    def chunked():
        for d, h in parts:
            d.copy_(h, non_blocking=True)
    print("H2D in %4d MB chunks %.1f GB/s" % (mb, timed([(s1, chunked)], 2)[0]))
