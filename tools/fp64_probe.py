"""FP64 issue-rate probes (DFMA / DMUL / DADD / mix), burst and sustained, with clocks."""
import ctypes, os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_00292_b200 as eig
L = eig.lib()
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
import bench  # noqa: E402
PR = bench.probes_lib()  # measurement probes: tools/probes/libeig33_probes.so (not the product)
PR.eig33_probe_fp64_op.restype = ctypes.c_double
PR.eig33_probe_fp64_op.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
import torch
torch.cuda.init()
for op, name in enumerate(["DFMA", "DMUL", "DADD", "MUL/ADD"]):
    burst = PR.eig33_probe_fp64_op(op, 10, 2048)
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    sus = PR.eig33_probe_fp64_op(op, 2000, 8192)
    p.terminate(); out = p.stdout.read().strip().splitlines()
    cl = [l for l in out if l.strip()][-5:]
    print(f"{name:8s} burst {burst/1e12:6.2f} T/s   sustained {sus/1e12:6.2f} T/s   clocks,power tail {cl}")
PR.eig33_probe_fp64_latency.restype = ctypes.c_double
PR.eig33_probe_fp64_latency.argtypes = [ctypes.c_int] * 3
for op, name in ((0, "DFMA"), (1, "DMUL"), (2, "DADD")):
    for ch in ((1, 2, 4, 8) if op == 0 else (1, 4)):
        for w in (1, 4, 8, 16):
            cyc = PR.eig33_probe_fp64_latency(op, ch, w)
            print(f"lat {name} chains={ch} warps/SM={w:2d}: {cyc:7.2f} cycles/iter -> {cyc/ch:6.2f} cyc/op/thread")
PR.eig33_probe_fp64_chaos.restype = ctypes.c_double
PR.eig33_probe_fp64_chaos.argtypes = [ctypes.c_double]
for secs in (0.05, 3.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    r = PR.eig33_probe_fp64_chaos(secs)
    p.terminate()
    out = [l for l in p.stdout.read().strip().splitlines() if l.strip()]
    print(f"chaotic DFMA {secs:4.2f} s: {r/1e12:6.2f} T/s   clocks/power tail {out[-3:]}")
