"""Throughput benchmark of the batched eig33 hot path (BASELINE.json metric:
3x3 fp64 eigvals/sec at 1/2/4/8 B200; % of HBM/FP64 roofline).

Workload (BASELINE configs[2], config 3): 2^28 general nonsymmetric records
A = (V diag(l)) V^-1, V Gaussian with cond2(V) <= 1e3, l ~ U[-10,10] -- 19.3 GB
in, 6.4 GB lambda out -- STRONG-sharded over the N GPUs exactly as SURVEY 8(e)
and the C++ host driver eig33_multi_eigvals cut a batch: rank r evaluates the
contiguous even-aligned shard shard_bounds(2^28, N, r).  A step = one
eig33cu_eigvals launch per rank over its shard; the step time is the max over
ranks (CUDA events on each rank's launch stream, all-gathered); value = 2^28 x
steps / that time.  No collective on the data path: torch.distributed carries
only the barrier and the timing/checksum reductions.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line on rank 0.  Besides the contract keys the line carries
  roofline        FP64 pipe and HBM for k_fused, both fractions, the binding one on top
  sustained       >= 3 s of back-to-back launches (time-blocked like the
                  reference's own perf loop, proj/src/bench.cpp:222-241), own clocks
  per_config      configs 1-5 at their BASELINE sizes, lambda and lambda+inv+flags
  e2e             the same batch through eig33_eigvals_host (pinned host buffers,
                  copies inside the timed region), one process per GPU
  multi_driver    the same batch through eig33_multi_eigvals from ONE process
                  over N devices (the north_star's host driver)
  cpu_baseline    the compiled reference core on this host (N=1 only)
--impl reference evaluates the same 2^28 records (host regeneration of the
counter-based corpus, bit-identical to the device generator: oracle/libcorpus.so)
with the compiled reference core (oracle/_ref) on all host cores.
"""
import argparse
import ctypes
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3×3 fp64 eigvals/sec at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "matrices/s"
N_TOTAL_DEFAULT = 1 << 28
SEED = 0x2511_00292
BYTES_PER_REC = 96          # 72 B in + 24 B lambda out
BYTES_PER_REC_FULL = 129    # + 32 B invariants + 1 B flags
BYTES_PER_REC_INV = 104     # invariants alone: 72 B in + 32 B out
FP64_OPS_PER_REC = 357      # frozen algorithmic FP64-pipe count
HBM_PEAK_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback
SPEC_FP64_INST_PER_S = 148 * 64 * 1.965e9  # 148 SMs x 64 FP64 lanes x max SM clock
CONFIG_SIZES = {1: 1 << 20, 2: 1 << 22, 3: 1 << 22, 4: 1 << 22, 5: 1 << 22}
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libeig33_ref.so")
CORPUS_SO = os.path.join(ROOT, "oracle", "libcorpus.so")
PROBES_SO = os.path.join(ROOT, "tools", "probes", "libeig33_probes.so")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1, help="GPUs (N>1: launch under torchrun, one rank each)")
    p.add_argument("--steps", type=int, default=20, help="timed steps (one launch per rank each)")
    p.add_argument("--warmup", type=int, default=5, help="untimed warm-up steps (>= 3)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"],
                   help="reference: the compiled reference core on all host cores (rank 0 only)")
    p.add_argument("--records", type=int, default=N_TOTAL_DEFAULT, help="records in the whole job (sharded over ranks)")
    p.add_argument("--e2e-steps", type=int, default=3, help="host-buffer (PCIe) end-to-end steps")
    p.add_argument("--sustained-seconds", type=float, default=3.0, help="length of the sustained sub-run (0: skip)")
    p.add_argument("--no-per-config", action="store_true", help="skip the configs 1-5 block")
    p.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end measurements")
    p.add_argument("--no-multi-driver", action="store_true", help="skip the single-process eig33_multi_eigvals leg")
    p.add_argument("--no-cpu-baseline", action="store_true", help="skip the CPU baseline leg (N=1 only anyway)")
    p.add_argument("--power-model", action="store_true",
                   help="also run the energy-model probes (idle / data path / stream / chaotic DFMA power)")
    p.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample length")
    p.add_argument("--dry-run", action="store_true",
                   help="CPU-only harness check (gloo, no kernels): sharding, timing reduction, JSON line")
    return p.parse_args()


def shard_of(n, world, rank):
    from paper_2511_00292_b200.shard import shard_bounds

    return shard_bounds(n, world, rank)


def config_block(n_total, world):
    """The workload description both arms print (identical dicts)."""
    return {
        "workload": "BASELINE config 3 (configs[2]): general nonsymmetric A=(V diag(l))V^-1, V~N(0,1) "
                    "with cond2(V)<=1e3, l~U[-10,10]; lambda-only output",
        "records_total": n_total,
        "records_per_gpu": [hi - lo for lo, hi in (shard_of(n_total, world, r) for r in range(world))],
        "sharding": "strong: contiguous even-aligned shards [2*floor(g*n/(2N)), ...) (SURVEY 8e)",
        "parallelism": f"dp{world} (contiguous shards, no collective)",
        "seed": SEED,
        "generator": "counter-based eig33_gen_core.h (device eig33cu_generate == host oracle/libcorpus.so, bitwise)",
        "l2": "inputs larger than L2 (19.3 GB per step at 2^28 records)",
    }


def host_description():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "libc": " ".join(platform.libc_ver()), "host_threads": os.cpu_count()}


# ---------------------------------------------------------------------------
# reference side (oracle/: the compiled reference core and the host corpus)
# ---------------------------------------------------------------------------
def ref_lib():
    """The compiled reference core; no fallback -- a missing build is an error."""
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(f"{REF_SO} missing: build it with `make -C oracle ref` where "
                                "/root/reference exists (it travels to the GPU box prebuilt)")
    L = ctypes.CDLL(REF_SO)
    P, S, I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    L.ref_eigvals.argtypes = [P, S, P, P, I]
    L.ref_checksum_loop.restype = ctypes.c_uint64
    L.ref_checksum_loop.argtypes = [P, ctypes.c_uint64]
    return L


def host_corpus(config, n, seed, first=0, threads=None):
    """Records [first, first+n) of a BASELINE config, regenerated on the host
    (bit-identical to eig33cu_generate)."""
    import numpy as np

    if not os.path.exists(CORPUS_SO):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
    C = ctypes.CDLL(CORPUS_SO)
    C.corpus_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_size_t,
                                  ctypes.c_void_p, ctypes.c_int]
    a = np.empty((n, 9))
    rc = C.corpus_generate(config, seed, first, n, a.ctypes.data, threads or os.cpu_count() or 1)
    if rc:
        raise RuntimeError("corpus_generate failed")
    return a


def checksum_u64(x):
    """Wrapping 64-bit sum of the records' bit patterns (numpy or torch)."""
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return int(x.view(torch.int64).sum().item()) & (2 ** 64 - 1)
    except ImportError:
        pass
    import numpy as np

    return int(x.view(np.uint64).sum(dtype=np.uint64))


def cpu_latency_ns(L, iterations=1_000_000):
    """The reference's own single-matrix latency discipline (src/bench.cpp:245-289):
    eigvals_checksum_loop on generate_case(D2, U1, 1e-14), 10 timed blocks after
    a warm-up block; returns (mean ns/eval, fastest ns/eval)."""
    import numpy as np

    from tests._util import perf_matrix

    m = np.ascontiguousarray(perf_matrix())
    reps, per = 10, iterations // 10
    L.ref_checksum_loop(m.ctypes.data, per // 10 + 1)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        L.ref_checksum_loop(m.ctypes.data, per)
        ts.append((time.perf_counter_ns() - t0) / per)
    return statistics.mean(ts), min(ts)


def cpu_eigvals_rate(L, a, seconds, threads):
    """Stream eig33::eigvals over the host sample `a` for ~`seconds` (>= 5 passes
    after a warm-up pass); returns (median-pass matrices/s, pass stats)."""
    import numpy as np

    n = a.shape[0]
    lam = np.empty((n, 3))

    def one():
        L.ref_eigvals(a.ctypes.data, n, lam.ctypes.data, None, threads)

    one()
    t0 = time.perf_counter()
    ts = []
    while True:
        t1 = time.perf_counter()
        one()
        ts.append(time.perf_counter() - t1)
        if time.perf_counter() - t0 >= seconds and len(ts) >= 5:
            break
    stats = {"passes": len(ts), "median": n / statistics.median(ts), "best": n / min(ts),
             "mean": n * len(ts) / sum(ts)}
    return n / statistics.median(ts), stats


def run_reference(args, rank, world):
    """The reference's own CPU implementation (the compiled, unmodified core) on
    every host core over the SAME 2^28 records the GPU arm evaluates; rank 0
    only, the other ranks exit without work."""
    if rank != 0:
        return
    import numpy as np

    threads = os.cpu_count() or 1
    n = args.records
    L = ref_lib()
    t0 = time.perf_counter()
    a = host_corpus(3, n, SEED, 0, threads)
    gen_s = time.perf_counter() - t0
    lam = np.empty((n, 3))

    def step():
        L.ref_eigvals(a.ctypes.data, n, lam.ctypes.data, None, threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    v = n * args.steps / el
    lat = cpu_latency_ns(L)
    cfg = config_block(n, world)
    cfg["input_checksum"] = f"{checksum_u64(a):016x}"
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"all {n} records of the GPU arm's batch (same seed, host regeneration "
                                   f"bit-identical to the device corpus) per step; eig33::eigvals "
                                   f"(oracle/_ref, the unmodified reference core) over contiguous shards "
                                   f"on {threads} threads",
                         "host_generation_s": gen_s,
                         "latency_ns": {"mean": lat[0], "fastest": lat[1],
                                        "loop": "eigvals_checksum_loop on generate_case(D2,U1,1e-14), "
                                                "10 x 1e5 evals"},
                         **host_description()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed regions)
# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler (100 ms) over the given GPUs; summaries cover the
    samples taken inside a named window [mark(name, start), mark(name, stop)]."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, devs):
        self.devs = list(devs)
        self.proc = None
        self.lines = []
        self.win = {}

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(map(str, self.devs)), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            time.sleep(0.3)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def begin(self, name):
        self.win[name] = [time.time(), None]

    def end(self, name):
        self.win[name][1] = time.time()

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, name):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0, t1 = self.win[name]
        sm, pw, mx, reasons = [], [], None, set()
        for ts, ln in list(self.lines):
            if not (t0 <= ts <= t1 + 0.1):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "power_w_median": statistics.median(pw) if pw else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "gpus": self.devs,
                "reasons": sorted(reasons)}

    def power_window(self, t0, t1):
        pw, sm = [], []
        for ts, ln in list(self.lines):
            f = [x.strip() for x in ln.split(",")]
            if t0 <= ts <= t1 and len(f) >= 4:
                try:
                    sm.append(float(f[1]))
                    pw.append(float(f[3]))
                except ValueError:
                    pass
        return (statistics.median(pw) if pw else None, statistics.median(sm) if sm else None)


# ---------------------------------------------------------------------------
# measurement helpers (GPU arm)
# ---------------------------------------------------------------------------
def probes_lib():
    """tools/probes/libeig33_probes.so: FP64 issue-rate and energy probes
    (measurement only; never part of the product library)."""
    if not os.path.exists(PROBES_SO):
        from paper_2511_00292_b200 import build

        build.build_probes()
    L = ctypes.CDLL(PROBES_SO)
    L.eig33_probe_fp64_rate.restype = ctypes.c_double
    L.eig33_probe_fp64_rate.argtypes = [ctypes.c_int]
    L.eig33_probe_fp64_chaos.restype = ctypes.c_double
    L.eig33_probe_fp64_chaos.argtypes = [ctypes.c_double]
    L.eig33_probe_stream.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p]
    L.eig33_probe_memonly.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]
    return L


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def ncu_traffic():
    """Per-record DRAM bytes of k_fused from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_k_fused.json")) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("records_per_launch")
    except (OSError, ValueError):
        return None, None


def roofline(rate_per_gpu, bytes_per_rec, hbm_peak, hbm_src, fp64_peak, fp64_src, ops=FP64_OPS_PER_REC):
    """Both roofs for one kernel at `rate_per_gpu` records/s; the binding roof
    (the slower one for this record mix) on top.  `ops` = algorithmic FP64
    instructions per record (0: an HBM-only kernel, the invariants alone)."""
    hbm_ach = rate_per_gpu * bytes_per_rec / 1e9
    fp64_ach = rate_per_gpu * ops / 1e12
    hbm = {"bound": "hbm", "achieved": hbm_ach, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_ach / hbm_peak,
           "peak_source": hbm_src, "bytes_per_record": bytes_per_rec}
    fp64 = {"bound": "fp64", "achieved": fp64_ach, "peak": fp64_peak, "unit": "T fp64-inst/s",
            "frac": fp64_ach / fp64_peak if fp64_peak else None, "peak_source": fp64_src,
            "frac_of_spec": fp64_ach * 1e12 / SPEC_FP64_INST_PER_S,
            "spec_peak": SPEC_FP64_INST_PER_S / 1e12,
            "ops_per_record": ops}
    binding = fp64 if (fp64["frac"] or 0) >= hbm["frac"] else hbm
    out = dict(binding)
    out["both"] = {"hbm": hbm, "fp64": fp64}
    return out


def time_launches(fn, stream, reps, torch):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def per_config_block(L, eig, torch, dev, stream, reps=20):
    """Configs 1-5 at their BASELINE sizes (config 3 at 2^22 here; its 2^28 is
    the headline): lambda only (96 B/record) and lambda + invariants + flags
    (129 B/record, what configs 1, 4 and 5 ask for); plus the other batched
    entry points on the config they fit: eigvalss with invariants and flags on
    the symmetric config 1 (src/eigensolver.cpp:97-117, 129 B/record) and the
    invariants alone on config 3 (src/invariants.cpp:76-98, 104 B/record,
    HBM-bound).  Burst rates: 20 launches each after 3 warm-ups, on a GPU that
    idled 0.5 s first."""
    out = {}
    for cfg, n in CONFIG_SIZES.items():
        with torch.cuda.stream(stream):
            a = eig.generate(cfg, n, seed=SEED + cfg, device=dev)
            lam = torch.empty((n, 3), dtype=torch.float64, device=dev)
            inv = torch.empty((n, 4), dtype=torch.float64, device=dev)
            fl = torch.empty((n,), dtype=torch.uint8, device=dev)
        stream.synchronize()
        pa, pl, pi, pf = (ctypes.c_void_p(x.data_ptr()) for x in (a, lam, inv, fl))
        st = ctypes.c_void_p(stream.cuda_stream)
        row = {"records": n}
        modes = [("lam", L.eig33cu_eigvals, (None, pl, None), BYTES_PER_REC, FP64_OPS_PER_REC),
                 ("lam_inv_flags", L.eig33cu_eigvals, (pi, pl, pf), BYTES_PER_REC_FULL, FP64_OPS_PER_REC)]
        if cfg == 1:  # symmetric: the reference's own entry point for it is eigvalss
            modes.append(("eigvalss_lam", L.eig33cu_eigvalss, (None, pl, None), BYTES_PER_REC, FP64_OPS_PER_REC))
            modes.append(("eigvalss_inv_flags", L.eig33cu_eigvalss, (pi, pl, pf), BYTES_PER_REC_FULL,
                          FP64_OPS_PER_REC))
        if cfg == 3:
            modes.append(("inv_only", L.eig33cu_invariants, (pi,), BYTES_PER_REC_INV, 0))
        for mode, entry, args_, bpr, ops in modes:
            def fn(entry=entry, args_=args_):
                rc = entry(pa, n, *args_, st)
                if rc:
                    raise RuntimeError(L.eig33cu_last_error().decode())
            time.sleep(0.5)
            for _ in range(3):
                fn()
            ms = time_launches(fn, stream, reps, torch)
            rate = n / (ms * 1e-3)
            row[mode] = {"value": rate, "unit": UNIT, "ms_per_launch": ms, "launches": reps,
                         "kernels_per_launch": 1,
                         "roofline": {"bytes_per_record": bpr, "ops_per_record": ops}}  # fractions: after the FP64 probe
        if cfg == 4 or cfg == 5:
            adv = int((fl.to(torch.int32) & 1).sum().item())
            row["advisory_share"] = adv / n
        out[str(cfg)] = row
        del a, lam, inv, fl
    return out


def pcie_rates(torch, h_a, h_l, dev):
    """Pinned-buffer copy rates (GB/s): H2D alone, D2H alone, H2D + D2H at once."""
    src = h_a.view(-1)[: min(h_a.numel(), 1 << 27)]
    out = h_l.view(-1)[: min(h_l.numel(), 1 << 27)]
    d_in = torch.empty(src.numel(), dtype=src.dtype, device=dev)
    d_out = torch.zeros(out.numel(), dtype=out.dtype, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(jobs, reps=3):
        torch.cuda.synchronize(dev)
        ev = []
        for s, f, nbytes in jobs:
            with torch.cuda.stream(s):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    f()
                e1.record()
                ev.append((e0, e1, nbytes))
        torch.cuda.synchronize(dev)
        return [reps * nb / (e0.elapsed_time(e1) * 1e-3) / 1e9 for e0, e1, nb in ev]

    h2d = (s1, lambda: d_in.copy_(src, non_blocking=True), src.numel() * 8)
    d2h = (s2, lambda: out.copy_(d_out, non_blocking=True), out.numel() * 8)
    timed([h2d], 1)
    r = {"h2d_gbs": timed([h2d])[0], "d2h_gbs": timed([d2h])[0]}
    r["h2d_concurrent_gbs"], r["d2h_concurrent_gbs"] = timed([h2d, d2h])
    del d_in, d_out
    return r


def power_model(P, clocks, pa, pl, n, st, stream, dev, torch):
    """Optional energy MODEL (--power-model).  It divides
    the board power limit by energy per record built from this kernel's own
    data path with the arithmetic removed (eig33_probe_memonly) plus 357 x the
    energy of a chaotic-operand DFMA -- a model partly defined by the kernel
    itself, reported as supporting evidence only, never as the roofline."""
    torch.cuda.synchronize()
    t = time.time()
    time.sleep(2.0)
    p_idle, _ = clocks.power_window(t + 1.0, time.time())

    def probe(fn, secs=2.5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        fn()
        e0.record(stream)
        t = time.time()
        k = 0
        while time.time() - t < secs:
            fn()
            k += 1
            if k % 16 == 0:
                stream.synchronize()
        e1.record(stream)
        e1.synchronize()
        w, mhz = clocks.power_window(t + 1.0, time.time())
        return k * n / (e0.elapsed_time(e1) * 1e-3), w, mhz

    dp_s, p_dp, mhz_dp = probe(lambda: P.eig33_probe_memonly(pa, n, pl, st))
    time.sleep(1.0)
    t = time.time()
    op_s = P.eig33_probe_fp64_chaos(2.5)
    p_fp64, mhz_fp64 = clocks.power_window(t + 1.0, time.time())
    if None in (p_idle, p_dp, p_fp64) or op_s <= 0:
        return None
    cap = 1000.0
    e_dp = (p_dp - p_idle) / dp_s
    e_op = (p_fp64 - p_idle) / op_s
    e_total = e_dp + FP64_OPS_PER_REC * e_op
    return {"kind": "model (self-referential: data-path term measured on this kernel with its "
                    "arithmetic removed); supporting evidence, not a roofline",
            "idle_w": p_idle, "limit_w": cap,
            "datapath": {"records_per_s": dp_s, "w": p_dp, "sm_mhz": mhz_dp, "nj_per_record": e_dp * 1e9},
            "fp64_chaos": {"inst_per_s": op_s, "w": p_fp64, "sm_mhz": mhz_fp64, "pj_per_inst": e_op * 1e12},
            "nj_per_record_model": e_total * 1e9,
            "model_records_per_s": (cap - p_idle) / e_total}


def bind_to_gpu_cpus(local_rank):
    """At N > 1: pin this rank's process to the CPUs NVML reports as local to
    its GPU (on a two-socket box, the GPU's own NUMA node), so the pinned host
    buffers of the e2e leg are allocated and copied on the socket whose PCIe root
    the GPU hangs off.  Returns the CPU count bound to, or None (NVML
    unavailable, single NUMA node: nothing changes)."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local_rank)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus and len(cpus) < len(os.sched_getaffinity(0)):
            os.sched_setaffinity(0, cpus)
        return len(cpus) or None
    except Exception:  # noqa: BLE001 -- a binding hint, never a failure
        return None


# ---------------------------------------------------------------------------
class HostSync:
    """Rank plumbing shared by the GPU arm and the dry run: the default process
    group (NCCL on the GPU arm, as the contract asks; gloo in the dry run) plus a
    gloo group that carries every host-side barrier and reduction -- an NCCL
    barrier would leave a spinning kernel on a waiting rank's GPU while rank 0
    drives all devices in the multi-driver leg."""

    def __init__(self, world, backend, device=None):
        self.world = world
        self.dist = self.pg = None
        if world > 1:
            import torch.distributed as dist

            if device is not None:
                dist.init_process_group(backend, device_id=device)
            else:
                dist.init_process_group(backend)
            self.dist = dist
            self.pg = dist.new_group(backend="gloo")

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier(group=self.pg)

    def gather(self, x):
        """all ranks' float x, in rank order"""
        if self.dist is None:
            return [float(x)]
        import torch

        t = torch.tensor([float(x)], dtype=torch.float64)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.pg)
        return [float(o.item()) for o in out]

    def gather_obj(self, x):
        if self.dist is None:
            return [x]
        out = [None] * self.world
        self.dist.all_gather_object(out, x, group=self.pg)
        return out

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2511_00292_b200 as eig

    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    bound_cpus = bind_to_gpu_cpus(local_rank) if world > 1 else None
    sync = HostSync(world, "nccl", dev)
    barrier, gather, gather_int = sync.barrier, sync.gather, sync.gather_obj

    L = eig.lib()
    P = probes_lib()
    n_total = args.records
    lo, hi = shard_of(n_total, world, rank)
    n = hi - lo
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        a = eig.generate(3, n, seed=SEED, first_index=lo, device=dev)
        lam = torch.empty((n, 3), dtype=torch.float64, device=dev)
    stream.synchronize()
    pa, pl = ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(lam.data_ptr())
    st = ctypes.c_void_p(stream.cuda_stream)
    # checksum of the whole job's records (wrapping 64-bit sum over ranks)
    input_checksum = sum(int(c) for c in gather_int(checksum_u64(a))) & (2 ** 64 - 1)

    def step():
        rc = L.eig33cu_eigvals(pa, n, None, pl, None, st)
        if rc:
            raise RuntimeError(L.eig33cu_last_error().decode())

    devs = list(range(world)) if rank == 0 else [local_rank]
    clocks = Clocks(devs if rank == 0 else [local_rank])
    clocks.start()

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    torch.cuda.synchronize()
    barrier()
    clocks.begin("headline")
    ms_rank = time_launches(step, stream, args.steps, torch) * args.steps
    clocks.end("headline")
    torch.cuda.synchronize()
    barrier()
    per_rank_ms = gather(ms_rank)
    ms_max = max(per_rank_ms)
    ms_step = ms_max / args.steps
    value = n_total * args.steps / (ms_max * 1e-3)

    # ---- sustained sub-run: time-blocked, >= args.sustained_seconds ----
    sustained = None
    if args.sustained_seconds > 0:
        time.sleep(0.5)
        barrier()
        clocks.begin("sustained")
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.time()
        k = 0
        while time.time() - t0 < args.sustained_seconds:
            for _ in range(8):
                step()
            k += 8
            stream.synchronize()
        e1.record(stream)
        e1.synchronize()
        clocks.end("sustained")
        ks = gather(k)
        mss = gather(e0.elapsed_time(e1))
        # each rank ran its own launch count; the job's step time is the slowest
        # rank's mean launch time
        ms_sus = max(m / kk for m, kk in zip(mss, ks))
        sustained = {"value": n_total / (ms_sus * 1e-3), "unit": UNIT, "seconds": max(mss) / 1e3,
                     "launches_per_rank": ks, "ms_per_step": ms_sus}
        barrier()

    # ---- e2e: the same shard through the public host-buffer API, pinned ----
    e2e = None
    h_a = h_l = None
    if not args.no_e2e:
        h_a = torch.empty((n, 9), dtype=torch.float64, pin_memory=True)
        h_a.copy_(a)
        h_l = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
        pha, phl = ctypes.c_void_p(h_a.data_ptr()), ctypes.c_void_p(h_l.data_ptr())
        rc = L.eig33_eigvals_host(pha, n, None, phl, None, local_rank)  # warm (staging alloc)
        if rc:
            raise RuntimeError(L.eig33cu_last_error().decode())
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            rc = L.eig33_eigvals_host(pha, n, None, phl, None, local_rank)
            if rc:
                raise RuntimeError(L.eig33cu_last_error().decode())
        el = time.perf_counter() - t0
        el_max = max(gather(el))
        same = bool(torch.equal(h_l.view(torch.int64), lam.cpu().view(torch.int64)))
        same_all = min(gather(1.0 if same else 0.0)) == 1.0
        link = pcie_rates(torch, h_a, h_l, dev)
        t_rec = 24 / link["d2h_concurrent_gbs"] + \
            max(0.0, 72 - link["h2d_concurrent_gbs"] * 24 / link["d2h_concurrent_gbs"]) / link["h2d_gbs"]
        model = 1e9 / t_rec
        e2e_value = n_total * args.e2e_steps / el_max
        e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n_total * 72,
               "d2h_bytes_per_step": n_total * 24, "steps": args.e2e_steps,
               "api": "eig33_eigvals_host per rank on its shard (pinned host buffers, chunked "
                      "H2D/kernel/D2H over 3 streams); wall clock, max over ranks",
               "bitwise_equal_to_device_path": same_all,
               "rank_cpu_binding": bound_cpus,
               "pcie_roofline": {"bound": "pcie", "h2d_gbs_measured": link["h2d_gbs"],
                                 "d2h_gbs_measured": link["d2h_gbs"],
                                 "concurrent_h2d_gbs": link["h2d_concurrent_gbs"],
                                 "concurrent_d2h_gbs": link["d2h_concurrent_gbs"],
                                 "duplex_model_records_per_s_per_gpu": model,
                                 "frac": e2e_value / world / model}}
        if world > 1:
            del h_a, h_l
            h_a = h_l = None
    barrier()

    # ---- power model (optional) ----
    pmodel = None
    if args.power_model and rank == 0:
        pmodel = power_model(P, clocks, pa, pl, n, st, stream, dev, torch)
        step()
        stream.synchronize()
    barrier()

    # ---- per-config block (rank 0; the others wait) ----
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs") or HBM_PEAK_FALLBACK
    hbm_src = "of measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else "of fallback"
    fp64_src_b = ("of builder-measured: burst DFMA issue rate on this GPU (tools/probes "
                  "eig33_probe_fp64_rate, 20 x 11 ms)")
    fp64_src_s = ("of builder-measured: sustained chaotic-operand DFMA rate on this GPU, 2.5 s "
                  "(tools/probes eig33_probe_fp64_chaos)")
    per_config = None
    if not args.no_per_config and rank == 0:
        per_config = per_config_block(L, eig, torch, dev, stream)
    barrier()

    # ---- multi-driver: one process, eig33_multi_eigvals over N devices ----
    multi = None
    if not args.no_e2e and not args.no_multi_driver:
        del a, lam
        torch.cuda.empty_cache()
        barrier()
        if rank == 0 and torch.cuda.device_count() < world:
            multi = {"skipped": f"rank 0 sees {torch.cuda.device_count()} devices, fewer than {world}"}
        elif rank == 0:
            if h_a is None:  # N>1: the whole batch on rank 0's host, pinned
                h_a = torch.empty((n_total, 9), dtype=torch.float64, pin_memory=True)
                h_l = torch.empty((n_total, 3), dtype=torch.float64, pin_memory=True)
                sl = 1 << 25
                for s0 in range(0, n_total, sl):
                    m = min(sl, n_total - s0)
                    h_a[s0:s0 + m].copy_(eig.generate(3, m, seed=SEED, first_index=s0, device=dev))
                torch.cuda.empty_cache()
            pha, phl = ctypes.c_void_p(h_a.data_ptr()), ctypes.c_void_p(h_l.data_ptr())
            rc = L.eig33_multi_eigvals(pha, n_total, None, phl, None, world)  # warm
            if rc:
                raise RuntimeError(L.eig33cu_last_error().decode())
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                rc = L.eig33_multi_eigvals(pha, n_total, None, phl, None, world)
                if rc:
                    raise RuntimeError(L.eig33cu_last_error().decode())
            el = time.perf_counter() - t0
            multi = {"value": n_total * args.e2e_steps / el, "unit": UNIT, "ngpu": world,
                     "steps": args.e2e_steps, "h2d_bytes_per_step": n_total * 72,
                     "d2h_bytes_per_step": n_total * 24,
                     "api": "eig33_multi_eigvals (one process, one host thread + stream set per device, "
                            "pinned host buffers); wall clock"}
        barrier()
    h_a = h_l = None

    # FP64 issue-rate peaks on this GPU (roofline denominators), measured last so
    # that their full-power DFMA does not precede the workload, each after 2 s
    # idle: burst (11 ms launches, for the short headline region and the
    # per-config launches) and sustained chaotic-operand DFMA over 2.5 s (for
    # the sustained sub-run)
    time.sleep(2.0)
    fp64_burst = P.eig33_probe_fp64_rate(20)
    fp64_sus = 0.0
    if args.sustained_seconds > 0:
        time.sleep(2.0)
        fp64_sus = P.eig33_probe_fp64_chaos(2.5)
    if per_config:
        for row in per_config.values():
            for mode in [k for k, v in row.items() if isinstance(v, dict) and "roofline" in v]:
                rf = roofline(row[mode]["value"], row[mode]["roofline"]["bytes_per_record"], hbm_peak, hbm_src,
                              fp64_burst / 1e12, fp64_src_b, ops=row[mode]["roofline"]["ops_per_record"])
                row[mode]["roofline"].update(bound=rf["bound"], frac=rf["frac"], frac_hbm=rf["both"]["hbm"]["frac"],
                                             frac_fp64=rf["both"]["fp64"]["frac"])

    clocks.stop()
    if rank != 0:
        sync.close()
        return

    per_gpu = value / world
    rf = roofline(per_gpu, BYTES_PER_REC, hbm_peak, hbm_src, fp64_burst / 1e12, fp64_src_b)
    traffic, recs = ncu_traffic()
    rf["traffic"] = traffic * n / recs if traffic and recs else None
    rf["traffic_source"] = "profiles/ncu_k_fused.json (ncu --set full, dram__bytes_read+write per record x records per launch)"
    rf["algorithmic_bytes_per_launch"] = n * BYTES_PER_REC
    rf["kernel"] = "k_fused<eigvals,TMA> (1 launch per step per rank)"
    if sustained:
        sustained["clocks"] = clocks.summary("sustained")
        sustained["roofline"] = roofline(sustained["value"] / world, BYTES_PER_REC, hbm_peak, hbm_src,
                                         fp64_sus / 1e12 if fp64_sus > 0 else None, fp64_src_s)
    if pmodel:
        rf["power_model"] = pmodel

    cpu = None
    if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
        Lr = ref_lib()
        threads = os.cpu_count() or 1
        samp = min(1 << 22, n_total)
        a_host = host_corpus(3, samp, SEED, 0, threads)
        rate, stats = cpu_eigvals_rate(Lr, a_host, args.cpu_seconds, threads)
        rate1, stats1 = cpu_eigvals_rate(Lr, a_host[: 1 << 20], min(args.cpu_seconds, 3.0), 1)
        lat = cpu_latency_ns(Lr)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
               "sample": f"first {samp} records of this run's config-3 batch (host regeneration, bitwise the "
                         f"same records), median of {stats['passes']} passes (~{args.cpu_seconds:.0f} s), "
                         f"eig33::eigvals (oracle/_ref) on {threads} threads",
               "passes": stats,
               "one_core": {"value": rate1, "unit": UNIT, "sample": f"first {1 << 20} records, "
                                                                  f"{stats1['passes']} passes on 1 thread"},
               "latency_ns": {"mean": lat[0], "fastest": lat[1],
                              "loop": "eigvals_checksum_loop on generate_case(D2,U1,1e-14), 10 x 1e5 evals"},
               **host_description()}

    cfg = config_block(n_total, world)
    cfg["input_checksum"] = f"{input_checksum:016x}"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "per_rank_ms": per_rank_ms,
        "roofline": rf,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "multi_driver": multi,
        "gpu_launches": args.steps,
        "clocks": clocks.summary("headline"),
        "sustained": sustained,
        "per_config": per_config,
        "fp64_probe_inst_per_s": {"burst": fp64_burst, "sustained": fp64_sus,
                                  "spec_at_max_clock": SPEC_FP64_INST_PER_S},
    }
    print(json.dumps(line), flush=True)
    sync.close()


def run_dry(args, rank, world):
    """CPU-only check of the N-rank harness (gloo): the same HostSync plumbing,
    shard of each rank, max-over-ranks timing reduction and JSON line shape as
    the GPU arm.  No kernel runs; the 'step' is a host sleep proportional to the
    rank's shard so rank times differ."""
    sync = HostSync(world, "gloo")
    lo, hi = shard_of(args.records, world, rank)
    sync.barrier()
    t0 = time.perf_counter()
    for _ in range(args.warmup + args.steps):
        time.sleep((hi - lo) * 1e-9)
    ms = (time.perf_counter() - t0) * 1e3 * args.steps / (args.warmup + args.steps)
    per = sync.gather(ms)
    shards = sync.gather_obj([lo, hi])
    cks = sync.gather_obj(rank + 1)
    sync.barrier()
    if rank == 0:
        print(json.dumps({"impl": "dry-run", "metric": METRIC, "value": args.records * args.steps / (max(per) * 1e-3),
                          "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": max(per) / args.steps, "higher_is_better": True, "scaling": "strong",
                          "per_rank_ms": per, "shards": shards, "rank_objects": cks,
                          "config": config_block(args.records, world)}),
              flush=True)
    sync.close()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        run_dry(args, rank, world)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
