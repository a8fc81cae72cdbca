import ctypes, os, statistics, subprocess, sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2511_00292_b200 as eig
L = eig.lib()
def sample(fn, secs=3.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3); t0 = time.time(); k = 0
    while time.time() - t0 < secs:
        fn(); k += 1
    torch.cuda.synchronize(); el = time.time() - t0; p.terminate()
    rows = [l.split(",") for l in p.stdout.read().strip().splitlines() if "," in l][6:]
    return statistics.median(float(r[0]) for r in rows), statistics.median(float(r[1]) for r in rows), k / el
n = 1 << 27
a = eig.generate(3, n, seed=1); lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
clk, pw, r = sample(lambda: L.eig33cu_eigvals(ctypes.c_void_p(a.data_ptr()), n, None, ctypes.c_void_p(lam.data_ptr()), None, ctypes.c_void_p(st)))
print(f"{os.environ.get('TAG','product'):8s} clk {clk:.0f} MHz power {pw:.0f} W  {r*n/1e9:.1f} G rec/s  -> {r*n*96/1e12:.2f} TB/s")
