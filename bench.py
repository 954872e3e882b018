"""Benchmark of the oblique-QR normal-equation hot path (oqr_normal) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--variant normal]
                    [--impl reference]

One step = one oqr_normal call (all of SURVEY.md s8(a): Z packing, fused Gram K1, slot reduction
K1r, Cholesky K2, triangular solve K3) on BASELINE.json configs[3] (m = 40000, n = 200; A is
12.8 GB > the 126 MB L2, so no L2 flush is needed between steps).  Prints ONE JSON line (rank 0).

value    = whole-job FP64 GFLOP/s with inputs resident in HBM, the paper's normalisation
           (2 m^2 n + 2 m n^2) / T.  N > 1 (torchrun): the same problem
           row-sharded over the ranks (strong scaling; one n x n all-gather per step; DESIGN.md
           s9), T = max over ranks.
e2e      = the same metric with pinned-host A, Z copied in and Q, R copied out every step.
roofline = the fused Gram kernel K1, timed live with CUDA events on the launching stream
           (liboqr's timing hook): achieved = 2 m^2 n flops / mean K1 launch time against the
           measured FP64 DMMA peak (tools/k0_probe.cu, profiles/).
cpu_baseline = the CPU oracle (oracle/, as it stands) on a bounded sample: the leading r x r
           principal block of the same A and the first r rows of Z.
--impl reference: the oracle itself timed as the reference arm (rank 0 only).
--sym: the NEXT-N4 symmetric family (block-lower triangle of A; own roofline).
--tridiag: the NEXT-N3 second workload (tridiagonal A, m = 100000, n = 200; paper normalisation
           2mn^2; roofline on the step's dominant kernel, K3 or K4t).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gen  # noqa: E402

FP64_DMMA_PEAK_TFLOPS = 37.2   # tools/k0_probe.cu on this pool's B200 (profiles/r01_k0_probe.txt)
PEAK_SOURCE = "measured: K0 DMMA m8n8k4 microbenchmark, sustained, profiles/r01_k0_probe.txt"
# BASELINE.json "metric", verbatim (tests/test_bench_contract.py checks it).  The roofline reported
# with it is the binding one of min(FP64 peak, HBM): at configs[3] the FP64 (DMMA) roof.
METRIC = "oblique-QR GFLOP/s (FP64, 1 B200) and % of min(FP64-peak, HBM) roofline vs CPU oracle"


def flops_paper(m, n):
    return 2.0 * m * m * n + 2.0 * m * n * n


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) while the timed region runs."""

    def __init__(self, dev_index: int, period: float = 0.005):
        self.dev_index, self.period = dev_index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.dev_index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {
                "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
                "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
                "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, bit in names.items():
                            if r & bit and k != "gpu_idle":
                                self.reasons.add(k)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            self.error = str(e)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


def cpu_model() -> str:
    try:
        return next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "?")
    except OSError:
        return "?"


def oracle_threads() -> int:
    """Host threads the oracle runs on: all cores of this process's affinity mask.  torchrun exports
    OMP_NUM_THREADS=1 to every rank; the oracle (rank 0 alone) is meant to use the whole host, so
    the variable is overridden before the oracle's OpenMP runtime loads."""
    t = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(t)
    try:  # already loaded (second call): set the runtime's count directly
        import ctypes
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(t)
    except OSError:
        pass
    return t


def cpu_oracle_sample(p, target_s: float = 12.0, lead=None):
    """Time the CPU oracle (as it stands) on the leading r x r principal block of the config's A
    and the first r rows of Z, with r sized for ~target_s of work.  Returns the cpu_baseline dict."""
    import oracle
    m, n = p.m, p.n
    threads = oracle_threads()

    def run(r):
        # the leading r x r principal block of A (lead(r) when this process holds only a row shard)
        A = np.ascontiguousarray(lead(r) if p.A is None else p.A[:r, :r])
        Z = np.ascontiguousarray(p.Z[:, :r])
        t = time.perf_counter()
        _, _, st = oracle.normal(A, Z, r)
        return time.perf_counter() - t, st

    r = min(m, 4096)
    dt, _ = run(r)
    rate = flops_paper(r, n) / dt
    # flops(r) ~ 2 r^2 n: pick r for ~target_s, in multiples of 64, capped at m
    r2 = int(min(m, max(r, math.sqrt(target_s * rate / (2.0 * n)))) // 64 * 64)
    if r2 > r:
        r = r2
        dt, _ = run(r)
    return {"value": flops_paper(r, n) / dt / 1e9, "unit": "GFLOP/s", "cores": threads,
            "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"oracle normal on the leading {r}x{r} principal block of the config's A and "
                      f"first {r} rows of Z (n={n}); {dt:.1f} s; OMP threads={threads}"}, r, dt


def oracle_protocol(configs):
    """SURVEY s8(d) CPU-oracle timing protocol (informational, not the driver's JSON line): each
    config's oracle oqr_normal, best of 3 (1 when a run exceeds 30 s), all host threads; c0 and c1
    also single-threaded; inputs generated outside the timed region.  Prints one JSON line per
    (config, threads)."""
    import oracle
    import ctypes
    oracle.build()
    model = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "?")
    allt = len(os.sched_getaffinity(0))
    for k in configs:
        p = gen.config(k)
        for threads in ([allt, 1] if k in (0, 1) else [allt]):
            os.environ["OMP_NUM_THREADS"] = str(threads)
            try:  # the oracle's OpenMP runtime is already loaded: set its thread count directly
                ctypes.CDLL("libgomp.so.1").omp_set_num_threads(threads)
            except OSError:
                pass
            best = float("inf")
            for _ in range(3):
                t = time.perf_counter()
                _, _, st = oracle.normal(p.A, p.Z, p.m)
                dt = time.perf_counter() - t
                best = min(best, dt)
                if dt > 30.0:
                    break
            print(json.dumps({"oracle": "normal", "config": k, "m": p.m, "n": p.n, "threads": threads,
                              "cpu": model, "best_s": best, "status": st,
                              "gflops": flops_paper(p.m, p.n) / best / 1e9}), flush=True)


def reference_arm(args, cfg, rank):
    if rank != 0:
        return
    oracle_threads()
    import oracle
    oracle.build()
    c = gen.CONFIGS[cfg]
    m, n = c["m"], c["n"]
    p = gen.config(cfg)
    base, r, _ = cpu_oracle_sample(p, target_s=6.0)
    A = np.ascontiguousarray(p.A[:r, :r])
    Z = np.ascontiguousarray(p.Z[:, :r])
    fn = oracle.VARIANTS[args.variant]
    for _ in range(args.warmup):
        fn(A, Z, r)
    t = time.perf_counter()
    for _ in range(args.steps):
        fn(A, Z, r)
    dt = (time.perf_counter() - t) / args.steps
    v = flops_paper(r, n) / dt / 1e9
    base.update(value=v)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"configs[{cfg}] oqr_{args.variant} m={m} n={n}; "
                                                    f"CPU oracle on leading {r}x{r} block",
                                        "m": m, "n": n},
        "cpu_baseline": base,
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_tridiag(args):
    """The paper's second workload (fig.perf-tridiag): A = tridiag(e, d, e),
    m = 100000, n = 200 (gen.TRIDIAG_CONFIGS["T"]), flops normalised 2 m n^2.  Roofline on the
    dominant kernel of the step -- the row substitution K3 or the tridiagonal Gram K4t (G = Z^T (T Z)
    on DMMA, Z read once with the stencil fused) -- timed live by the hook."""
    import torch
    import oracle
    import paper_1401_5171_b200 as oqr
    d, e, p = gen.tridiag_config("T")
    m, n = p.m, p.n
    fl = 2.0 * m * n * n
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    d_h, e_h, Z_h = torch.from_numpy(d).pin_memory(), torch.from_numpy(e).pin_memory(), torch.from_numpy(p.Z)
    Z_h = Z_h.pin_memory()
    dg, eg, Z = d_h.to(dev), e_h.to(dev), Z_h.to(dev)
    Q = torch.empty((n, m), dtype=torch.float64, device=dev)
    R = torch.empty((n, n), dtype=torch.float64, device=dev)
    Q_h = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
    R_h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    fn = oqr.VARIANTS_TRIDIAG[args.variant]
    for _ in range(args.warmup):
        assert fn(dg, eg, Z, Q, R)[2] == 0
    # the timed region: the synchronous call as a user makes it (from its second identical call on
    # the library replays a cached CUDA graph of the step, include/oqr.h)
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sts = [fn(dg, eg, Z, Q, R)[2] for _ in range(args.steps)]
        e1.record(stream)
        torch.cuda.synchronize()
    assert all(st == 0 for st in sts), sts
    ms_step = e0.elapsed_time(e1) / args.steps
    # per-kernel times: the same steps again with the library's per-kernel CUDA-event hook (on the
    # launching stream); the hook bypasses the graph cache, so this pass runs the direct path
    oqr.timing_enable(True)
    oqr.timing_reset()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        assert fn(dg, eg, Z, Q, R)[2] == 0
    torch.cuda.synchronize()
    kern = {k: oqr.timing_read_kernel(k) for k in ("K4", "K3", "K2")}
    _, _, launches = oqr.timing_read()
    oqr.timing_enable(False)
    k4_ms = kern["K4"][0] / max(kern["K4"][1], 1)
    k3_ms = kern["K3"][0] / max(kern["K3"][1], 1)
    NT = (n + 7) // 8
    # The roofline goes on the dominant kernel of the step (the larger mean launch time):
    #   K4t computes the upper triangle only (G is symmetric): its algorithmic work is the upper
    #   8 x 8 tiles incl. the diagonal ones, 2 m 64 NT (NT + 1) / 2 flops (Z read once: 8mn bytes);
    #   K3 (Q = Z R^{-1}, row substitution): m n^2 flops, 16 m n bytes (Z in, Q out) -- tensor-bound
    #   at n = 200 (m n^2 / P = 108 us > 16 m n / B = 49 us)
    fl_k4 = 2.0 * m * 64 * NT * (NT + 1) / 2
    fl_k3 = 1.0 * m * n * n
    if k3_ms > k4_ms:
        dom, dom_ms, dom_fl = "K3", k3_ms, fl_k3
        dom_name = "trsm (K3): Q = Z R^{-1} row substitution, off-diagonal tiles on DMMA"
        traffic_file = "k3_tridiag_traffic.json"
    else:
        dom, dom_ms, dom_fl = "K4", k4_ms, fl_k4
        dom_name = "gram_tridiag (K4t, Z read once by TMA, stencil fused): upper triangle of G = Z^T (T Z)"
        traffic_file = "k4_tridiag_traffic.json"
    achieved = dom_fl / (dom_ms * 1e-3) / 1e12
    # e2e: d, e, Z in from pinned host memory, Q, R out, every step
    h2d = (d_h.numel() + e_h.numel() + Z_h.numel()) * 8
    d2h = (Q_h.numel() + R_h.numel()) * 8
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.e2e_steps):
        dg.copy_(d_h, non_blocking=True)
        eg.copy_(e_h, non_blocking=True)
        Z.copy_(Z_h, non_blocking=True)
        Qs, Rs, st = fn(dg, eg, Z, Q, R)
        Q_h.copy_(Qs, non_blocking=True)
        R_h.copy_(Rs, non_blocking=True)
        assert st == 0
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_value = fl / (e0.elapsed_time(e1) / args.e2e_steps * 1e-3) / 1e9
    cpu = None
    if not args.no_cpu_baseline:   # the oracle on the leading mc rows (a tridiagonal of size mc)
        threads = oracle_threads()
        mc = m          # the whole problem takes well under a second on the host
        Zc = np.ascontiguousarray(p.Z[:, :mc])
        t = time.perf_counter()
        _, _, sto = oracle.VARIANTS_TRIDIAG[args.variant](d[:mc], e[:mc - 1], Zc, mc)
        dt = time.perf_counter() - t
        cpu = {"value": 2.0 * mc * n * n / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"oracle {args.variant}_tridiag on the leading {mc} rows (tridiagonal of size {mc}, "
                         f"n={n}); {dt:.1f} s; OMP threads={threads}"}
    traffic = None
    tp = os.path.join(ROOT, "profiles", traffic_file)
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            pass
    line = {
        "metric": "oblique-QR GFLOP/s, tridiagonal A (FP64, 1 B200; paper normalisation 2mn^2)",
        "value": fl / (ms_step * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"tridiag T oqr_{args.variant}_tridiag: m={m}, n={n}, kappa_A=1e3, kappa_Z=1e2",
                   "m": m, "n": n, "variant": args.variant, "flops_per_step": fl,
                   "flop_normalisation": "2mn^2 (PAPER.md:960-961)",
                   "l2": "Z = %.0f MB, Q = %.0f MB > L2; no flush" % (8e-6 * m * n, 8e-6 * m * n)},
        "roofline": {"bound": "tensor",
                     "kernel": dom_name,
                     "achieved": achieved,
                     "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_DMMA_PEAK_TFLOPS,
                     "traffic": traffic, "algorithmic_flops_per_launch": dom_fl, "mean_launch_ms": dom_ms,
                     "share_of_step": dom_ms / ms_step, "peak_source": PEAK_SOURCE,
                     "other_kernels_ms": {k: v for k, v in {
                         "gram_tridiag (K4t)": k4_ms, "trsm (K3)": k3_ms,
                         "potrf (K2)": kern["K2"][0] / max(kern["K2"][1], 1)}.items()
                         if not k.endswith("(%s)" % ("K4t" if dom == "K4" else dom))},
                     "kernel_times": "second pass of the same steps with the per-kernel event hook (direct path, K2 and K3 one after the other; the timed steps run them overlapped)",
                     "k4t_frac": fl_k4 / (k4_ms * 1e-3) / 1e12 / FP64_DMMA_PEAK_TFLOPS,
                     "k3_frac": fl_k3 / (k3_ms * 1e-3) / 1e12 / FP64_DMMA_PEAK_TFLOPS},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": args.e2e_steps, "api": f"H2D copies + oqr_{args.variant}_tridiag + D2H copies"},
        "gpu_launches": launches,   # the hook pass's count: the same kernels the replayed graph runs
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


_registered = []


def pinned(shape):
    """Page-locked float64 host tensor (numpy buffer + cudaHostRegister: no power-of-two
    rounding of torch's pinned caching allocator for the 12.8 GB A)."""
    import torch
    a = np.empty(shape, dtype=np.float64)
    rc = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister failed ({rc})")
    _registered.append(a)
    t = torch.from_numpy(a)
    assert t.is_pinned()
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--variant", default="normal", choices=["normal", "normal2", "prequr", "prequr_hh"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--oracle-protocol", default=None, metavar="CONFIGS",
                    help="SURVEY s8(d) CPU-oracle timing for the given configs (e.g. 0,1,4,2,3) and exit")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sym", action="store_true",
                    help="NEXT-N4 symmetric family: block-lower triangle of A only (own roofline)")
    ap.add_argument("--tridiag", action="store_true",
                    help="NEXT-N3 second workload: A tridiagonal, m = 100000, n = 200 (paper's 2mn^2 "
                         "normalisation, roofline on the step's dominant kernel)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the row-sharded code path even at N = 1 (it is the default for N > 1)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl != "reference":
        # allowed (e.g. for an ncu launch list), but such a line is not a valid measurement
        print(f"bench.py: --warmup {args.warmup} < 3: the timing rules need at least 3 warm-up steps",
              file=sys.stderr)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` outside torchrun: launch the N ranks ourselves (one process per
        # GPU, torch.distributed.run on 127.0.0.1); never measure 1 GPU under an N-GPU label
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        print("bench.py: launching " + " ".join(cmd), file=sys.stderr, flush=True)
        os.execv(sys.executable, cmd)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to report a mislabelled line",
              file=sys.stderr)
        sys.exit(2)
    if args.oracle_protocol is not None:
        if rank == 0:
            oracle_protocol([int(c) for c in args.oracle_protocol.split(",")])
        return
    if args.impl == "reference":
        reference_arm(args, args.config, rank)
        return
    if args.tridiag:
        assert world == 1, "--tridiag is a single-GPU workload"
        bench_tridiag(args)
        return

    import torch
    import torch.distributed as dist
    import paper_1401_5171_b200 as oqr

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or (args.sharded and "RANK" in os.environ):  # torchrun: the NCCL exchange runs
        dist.init_process_group("nccl", device_id=dev)
    c = gen.CONFIGS[args.config]
    m, n = c["m"], c["n"]
    fl = flops_paper(m, n)
    stream = torch.cuda.current_stream()
    Z_h = pinned((n, m))
    if world == 1 and not args.sharded:
        # inputs: generated once on the host straight into pinned buffers, then copied to HBM
        A_h = pinned((m, m))
        p = gen.config(args.config, A_out=A_h.numpy(), Z_out=Z_h.numpy())
        r0, mr = 0, m
        Q_h = pinned((n, m))
        fn = (oqr.VARIANTS_SYM if args.sym else oqr.VARIANTS)[args.variant]
        Q = torch.empty((n, m), dtype=torch.float64, device=dev)
        R = torch.empty((n, n), dtype=torch.float64, device=dev)

        def step(A, Z):
            Qo, Ro, st = fn(A, Z, Q, R)
            return Qo, Ro, st
    else:
        # row-sharded strong scaling: this rank generates and holds only its rows
        from paper_1401_5171_b200.dist import VARIANTS_ROWS, row_partition
        assert not args.sym, "the row-sharded path streams the dense row blocks of A"
        rows_fn = VARIANTS_ROWS[args.variant]
        r0, mr = row_partition(m, world)[rank]
        ldar = mr + (mr & 1)
        A_h = pinned((m, ldar))
        gen.config_A_rows(args.config, r0, r0 + mr, lda=ldar, out=A_h.numpy())
        p = gen.config(args.config, with_A=False, Z_out=Z_h.numpy())
        Q_h = pinned((n, mr))

        def step(A, Z):
            return rows_fn(A, Z, r0, mr)
    fl_gram = 2.0 * mr * m * n  # per K1 launch on this rank
    if args.sym:  # block-lower triangle incl. the 64 x 64 diagonal panels
        fl_gram = 2.0 * n * sum(min(64, m - i0) * min(m, i0 + 64) for i0 in range(0, m, 64))
    A = A_h.to(dev)
    Z = Z_h.to(dev)
    R_h = pinned((n, n))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        _, _, st = step(A, Z)
        assert st == 0, f"warm-up status {st}: {oqr.status_string(st)}"

    # ---- timed region: inputs resident in HBM ----
    oqr.timing_enable(True)
    oqr.timing_reset()
    statuses = []
    barrier()
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            statuses.append(step(A, Z)[2])
        e1.record(stream)
        barrier()
    ms_total = e0.elapsed_time(e1)
    gram_ms, gram_launches, launches = oqr.timing_read()
    other_ms = {}
    for kname, label in (("K2", "potrf (K2)"), ("K3", "trsm (K3)"), ("K4", "packed / tridiagonal Gram (K4', K4t)"), ("K6", "hhqr (K6)")):
        kms, kl = oqr.timing_read_kernel(kname)
        if kl:
            other_ms[label] = kms / kl
    oqr.timing_enable(False)
    assert all(s == 0 for s in statuses), statuses
    t_local = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_step = float(t_local.item()) / args.steps
    value = fl / (ms_step * 1e-3) / 1e9  # the whole problem, all ranks

    # ---- end to end through the public call with host buffers ----
    h2d = A_h.numel() * 8 + Z_h.numel() * 8
    if args.sym:
        h2d = sum((m - j0) * min(64, m - j0) for j0 in range(0, m, 64)) * 8 + Z_h.numel() * 8
    d2h = Q_h.numel() * 8 + R_h.numel() * 8
    # single-GPU dense CHOLQR: the host-array call, which overlaps the A transfer with the Gram
    host_call = world == 1 and not args.sharded and not args.sym and args.variant == "normal"
    e2e_api = ("oqr_normal_host (A staged in column chunks, H2D overlapped with K1)" if host_call else
               ("oqr_upload_sym + " if args.sym else "H2D copies + ") + f"oqr_{args.variant} + D2H copies")
    if host_call:
        _, _, st = oqr.normal_host(A_h, Z_h, Q_h, R_h)   # warm-up: pool allocation of the device A
        assert st == 0, st
    barrier()
    e0.record(stream)
    for _ in range(args.e2e_steps):
        if host_call:
            _, _, st = oqr.normal_host(A_h, Z_h, Q_h, R_h)
            assert st == 0
            continue
        if args.sym:
            oqr.upload_sym(A_h, A)      # only the block-lower triangle the *_sym calls read
        else:
            A.copy_(A_h, non_blocking=True)
        Z.copy_(Z_h, non_blocking=True)
        Qs, Rs, st = step(A, Z)
        Q_h.copy_(Qs, non_blocking=True)
        R_h.copy_(Rs, non_blocking=True)
        assert st == 0
    e1.record(stream)
    barrier()
    t_e2e = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = fl / (float(t_e2e.item()) * 1e-3) / 1e9

    if rank == 0:
        k1_ms = gram_ms / max(gram_launches, 1)
        achieved = fl_gram / (k1_ms * 1e-3) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "k1_traffic.json")
        if os.path.exists(tp):
            try:
                t = json.load(open(tp))
                if t.get("m") == m and t.get("n") == n and world == 1 and not args.sharded:
                    traffic = t["sym" if args.sym else "dense"]["dram_bytes_per_launch"]
            except Exception:
                pass
        cpu = None
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N = 1 only
            cpu, _, _ = cpu_oracle_sample(
                p, lead=lambda r: gen.config_A_rows(args.config, 0, r)[:r, :r])
        peaks = measured_peaks()
        line = {
            # --sym: the symmetric schedule does about half the dense flops; its value is the dense
            # problem's flops over its time (DENSE-EQUIVALENT rate, can exceed the FP64 peak), so it
            # is not reported under BASELINE's metric string
            "metric": METRIC if not args.sym else
            "oblique-QR dense-equivalent GFLOP/s, symmetric-half A (FP64, 1 B200; 2m^2n+2mn^2 over the time "
            "of the block-lower-triangle algorithm)",
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"configs[{args.config}] oqr_{args.variant}{'_sym' if args.sym else ''}: m={m}, n={n}, "
                                   f"kappa_A={c['kappa_a']:g}, kappa_Z={c['kappa_z']:g}",
                       "m": m, "n": n, "variant": args.variant,
                       "flops_per_step": fl,
                       "flop_normalisation": ("dense-equivalent: 2m^2n+2mn^2 (PAPER.md:959-961) although the "
                                              "symmetric schedule performs ~m^2n+2mn^2") if args.sym else
                       "2m^2n+2mn^2 (PAPER.md:959-961)",
                       "l2": "inputs (A = %.1f GB) larger than L2; no flush" % (8 * m * m / 1e9),
                       "parallelism": (f"row-sharded x{world}: one n x n all-gather per step (NCCL), "
                                       "fixed rank-order sum") if (world > 1 or args.sharded) else "single GPU"},
            "roofline": {"bound": "tensor",
                         "kernel": "gram_fused (K1)" + (" symmetric schedule: block-lower triangle" if args.sym else ""),
                         "achieved": achieved,
                         "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_DMMA_PEAK_TFLOPS, "traffic": traffic,
                         "algorithmic_flops_per_launch": fl_gram, "mean_launch_ms": k1_ms,
                         "share_of_step": k1_ms * gram_launches / args.steps / ms_step, "peak_source": PEAK_SOURCE,
                         "hbm_gbs_measured": peaks.get("hbm_gbs"),
                         "other_kernels_mean_launch_ms": other_ms},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": args.e2e_steps, "api": e2e_api},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
