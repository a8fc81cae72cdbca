"""Die-locality energy experiment (research, not product): see die_probe.cu.
  python tools/die_probe/run.py      (builds libdie_probe.so if missing)"""
import ctypes, os, statistics, subprocess, sys, time
import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libdie_probe.so")
if not os.path.exists(SO):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                    "-fPIC", "-o", SO, os.path.join(HERE, "die_probe.cu")], check=True)
D = ctypes.CDLL(SO)
P = lambda t: ctypes.c_void_p(t.data_ptr())
GRAN = 2048
NG = (4 << 30) // GRAN  # 4 GiB buffer
buf = torch.randint(-2 ** 62, 2 ** 62, (NG * GRAN // 8,), dtype=torch.int64, device="cuda")  # random bits
assert D.dp_init_self(P(buf), ctypes.c_longlong(NG), GRAN // 8) == 0
sms = torch.cuda.get_device_properties(0).multi_processor_count

# 1. SM clustering
M, B = 64, sms * 4
sm_out = torch.zeros(B, dtype=torch.int32, device="cuda")
lat = torch.zeros(B * M, dtype=torch.int32, device="cuda")
assert D.dp_sm_lat(P(buf), B, M, GRAN // 8, 3, P(sm_out), P(lat)) == 0
sm_of = sm_out.cpu().numpy()
L = lat.cpu().numpy().reshape(B, M)
per_sm = np.full((sms, M), 1 << 30)
for b in range(B):
    per_sm[sm_of[b]] = np.minimum(per_sm[sm_of[b]], L[b])
print("L2-hit latency per SM (cycles): min", per_sm.min(), "median", int(np.median(per_sm)), "max", per_sm.max())
# near/far pattern of each SM over the M granules (below the per-granule median = near);
# SMs on one die share the pattern, the other die has its complement
pat = per_sm < np.median(per_sm, axis=0, keepdims=True)
same = (pat == pat[0]).mean(axis=1)
A = same > 0.5
print(f"SM split: {A.sum()} / {(~A).sum()} SMs; pattern agreement with SM0's side: "
      f"same-die min {same[A].min():.3f}, other-die max {same[~A].max():.3f}")

# 2. granule map from die-A SMs
mask = np.zeros(8, np.uint32)
for s in np.nonzero(A)[0]:
    mask[s >> 5] |= np.uint32(1 << (s & 31))
mask_t = torch.from_numpy(mask.view(np.int32)).cuda()
glat = torch.zeros(NG, dtype=torch.int32, device="cuda")
done = torch.zeros(1, dtype=torch.int64, device="cuda")
t0 = time.time()
assert D.dp_granule_lat(P(buf), ctypes.c_longlong(NG), GRAN // 8, P(mask_t), P(glat), P(done), sms) == 0  # 1 warp/SM: no queueing
gl = glat.cpu().numpy()
thr_g = (np.percentile(gl, 5) + np.percentile(gl, 95)) / 2
nearA = np.nonzero(gl < thr_g)[0].astype(np.int64)
nearB = np.nonzero(gl >= thr_g)[0].astype(np.int64)
print(f"granule map in {time.time() - t0:.1f} s: near-A {len(nearA)}, near-B {len(nearB)}; "
      f"latency p5 {np.percentile(gl, 5):.0f} p50 {np.percentile(gl, 50):.0f} p95 {np.percentile(gl, 95):.0f}")

# 3. stream energy: near / far / mixed assignment
die_of_sm = torch.from_numpy((~A).astype(np.int32)).cuda()  # die 0 = A
rng = np.random.default_rng(0)


def sample(l0, l1, secs=3.0):
    t_l0, t_l1 = torch.from_numpy(l0).cuda(), torch.from_numpy(l1).cuda()
    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def one():
        ctr.zero_()
        D.dp_stream_sel(P(buf), GRAN, P(die_of_sm), P(t_l0), P(t_l1), ctypes.c_longlong(len(l0)),
                        ctypes.c_longlong(len(l1)), P(ctr), P(out), sms * 2, st)
    one()
    torch.cuda.synchronize()
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    k = 0
    t = time.time()
    while time.time() - t < secs:
        one()
        k += 1
        if k % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    p.terminate()
    rows = [ln.split(",") for ln in p.stdout.read().strip().splitlines() if "," in ln][6:]
    w = statistics.median(float(r[1]) for r in rows)
    mhz = statistics.median(float(r[0]) for r in rows)
    gbs = k * (len(l0) + len(l1)) * GRAN / (e0.elapsed_time(e1) * 1e-3) / 1e9
    return gbs, w, mhz


n = min(len(nearA), len(nearB))
a_, b_ = nearA[:n], nearB[:n]
mixed = rng.permutation(np.concatenate([a_, b_]))
for name, l0, l1 in (("near", a_, b_), ("far", b_, a_), ("mixed", mixed[:n], mixed[n:]),
                     ("near", a_, b_), ("far", b_, a_)):
    gbs, w, mhz = sample(l0, l1)
    print(f"{name:6s} read {gbs:7.0f} GB/s  {w:6.0f} W  {mhz:5.0f} MHz  -> {(w - 258) / gbs * 1e3:6.1f} pJ/B above idle")
