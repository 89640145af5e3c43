#!/usr/bin/env python3
"""bench.py -- fp64 tiled-QR throughput on B200 (BASELINE.json metric).

One step = the whole hot path on one matrix already resident
in HBM: pack A into tiles (a1), the DAG-executed factorization GEQRT/TSQRT/LARFB/SSRFB
(a2-a6, one persistent launch), and R extraction (a7).  value = standard flops
2mn^2 - 2n^3/3 per step / step time, summed over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl tqr|reference]

N > 1 (torchrun): ONE matrix factored by all ranks (strong scaling):
tile columns 1D block-cyclic, the panel tasks store packed V/T into every rank's workspace
over NVLink peer memory (CUDA IPC, exchanged once through torch.distributed).  Timing:
CUDA events on the plan's stream, barrier + synchronize on both sides, max over ranks.
Inputs (2 GiB at C3) exceed L2 (126 MB), so no flush is needed between steps.

--impl reference times the CPU oracle (oracle/, the deliberately plain C implementation
of the same algorithm) as it stands on the host cores, on a bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import tqr_inputs  # noqa: E402

METRIC = "fp64 tiled-QR GFLOP/s (2mn²−2n³/3) and % of fp64 peak at 1/2/4/8 B200"
# fp64 DMMA.8x8x4 peak measured on this pool's B200 (tools/probe_fp64.cu, profiles/r01_m0_fp64_probe.txt):
# 37.14 TFLOP/s = 148 SM x 64 FMA/clk x 2 x 1.965 GHz (99.8% of nominal).  MEASURED_PEAKS.json has no
# fp64 entry; this is our own measurement of the same pipe.
FP64_PEAK_TFLOPS = 37.14
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(tqr_inputs.CONFIGS))
    ap.add_argument("--impl", default="tqr", choices=["tqr", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--trace", default="", help="write a per-task execution trace (JSON) of one extra step")
    ap.add_argument("--method", default="qr", choices=["qr", "lu"],
                    help="lu: the tiled LU (include/tlu.h, SURVEY NEXT-4) on the config's matrix, 1 GPU")
    ap.add_argument("--schedule", default="critical", choices=["critical", "locality"],
                    help="locality: TQR_FLAG_LOCALITY dispatch order (DESIGN.md R22)")
    ap.add_argument("--tiles", default="square", choices=["square", "2bxb"],
                    help="2bxb: the paper's non-square 2b x b tiles (TQR_FLAG_TALL_TILES, DESIGN.md R30)")
    ap.add_argument("--emulate-ranks", type=int, default=1,
                    help="test mode: run the G-rank distributed schedule in one launch on one GPU")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.samples, self.stop = gpu, [], threading.Event()
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 4 + i and s[4 + i] == "Active"})
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "power_w_max": max(pw) if pw else None, "samples": len(self.samples)}


FULL_ORACLE_MAX_FLOPS = 1.2e13   # C1-C4: the whole workload (C3 ~80 s on 16 host threads); C5 (3.8e14): a sample


def sample_block(cfg, A=None):
    """A bounded sample of the workload's OWN bytes: the leading principal submatrix (same
    tiling, same seeded entries) -- 6144^2 for the square configs, 32 x 4 tiles for C4."""
    b = cfg["b"]
    m = n = min(cfg["m"], cfg["n"], max(8 * b, 6144 // b * b))
    if cfg["m"] > 4 * cfg["n"]:  # tall-skinny: keep the aspect ratio class
        n = min(cfg["n"], 4 * b)
        m = min(cfg["m"], 32 * n)
    if A is None:
        A = tqr_inputs.make(cfg["m"], cfg["n"], cfg["dist"], cfg["seed"])
    return np.asfortranarray(A[:m, :n])


def time_oracle(A, cfg, threads, h=1):
    """The oracle as it stands (oracle/, plain C DAG executor) on host matrix A (h = 2: its
    2b x b tile mode).  Returns (GFLOP/s standard count, seconds, tiles At, T)."""
    import oracle
    m, n = A.shape
    t0 = time.perf_counter()
    At, T = oracle.geqrf(A, cfg["b"], cfg["s"], nthreads=threads, h=h)
    dt = time.perf_counter() - t0
    return oracle.flops_standard(m, n) / dt / 1e9, dt, At, T


def run_reference(args, cfg, rank):
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    vals = []
    S = sample_block(cfg)
    desc = (f"oracle_geqrf_tiles on the leading {S.shape[0]}x{S.shape[1]} block of the {cfg['m']}x{cfg['n']} "
            f"workload matrix (same seeded bytes, b={cfg['b']} s={cfg['s']}), {threads} threads, one "
            f"factorization per step")
    for it in range(args.warmup + args.steps):
        v, dt, _, _ = time_oracle(S, cfg, threads)
        if it >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "m": cfg["m"], "n": cfg["n"], "b": cfg["b"], "s": cfg["s"],
                       "sample": desc},
            "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


LU_METRIC = "fp64 tiled-LU GFLOP/s (mn\u00b2\u2212n\u00b3/3) and % of fp64 peak"
LU_FULL_ORACLE_MAX_FLOPS = 2.0e11


def lu_property_parity(At_g, Wg, piv_g, U_g, A_host, b, s, threads, tile_cols):
    """DESIGN.md LU10: max |multiplier| and |Ltilde| (<= 1 for partial pivoting in the GPU's own
    arithmetic) and the backward error of the recorded transformation M (the oracle's replay from
    the GPU's factors) on A's tile columns `tile_cols` (None: all), in units of n u ||A||_max rho."""
    import oracle
    m, n = A_host.shape
    p_, q_ = -(-m // b), -(-n // b)
    K_ = min(p_, q_)
    T_g = At_g.reshape(q_, p_, b, b)
    mx = max(max(float(np.max(np.abs(np.tril(T_g[k, k].T, -1)))) for k in range(K_)),
             max((float(np.max(np.abs(T_g[k, k + 1:]))) for k in range(K_) if k + 1 < p_), default=0.0))
    Lt_g = np.zeros_like(Wg)
    for k in range(K_):
        for i in range(k + 1, p_):
            sl_ = (i + k * p_) * s * b
            for c0 in range(0, b, s):
                Wl = Wg[sl_ + c0 * s: sl_ + (c0 + s) * s].reshape(s, s, order="F")
                Lt_g[sl_ + c0 * s: sl_ + (c0 + s) * s] = (np.linalg.inv(Wl) - np.eye(s)).reshape(-1, order="F")
    cols = np.arange(n) if tile_cols is None else np.concatenate(
        [np.arange(j * b, min(n, (j + 1) * b)) for j in tile_cols])
    MA = oracle.lu_apply(At_g, Lt_g, piv_g, m, n, b, s, np.asfortranarray(A_host[:, cols]), nthreads=threads)
    kk = min(m, n)
    rho = max(1.0, float(np.max(np.abs(U_g)) / np.max(np.abs(A_host))))
    res = float(np.max(np.abs(MA[:kk] - U_g[:, cols])))
    if m > kk:
        res = max(res, float(np.max(np.abs(MA[kk:]))))
    be = res / (max(m, n) * 2.0 ** -53 * float(np.max(np.abs(A_host))) * rho)
    lt = float(np.max(np.abs(Lt_g)))
    return {"max_abs_multiplier": mx, "max_abs_ltilde": lt, "growth_rho": rho, "backward_error_n_u_rho": be,
            "ok": mx <= 1.0 and lt <= 1.0 + 1e-12 and be < 1.0}


def run_lu(args, cfg, rank, world, local):
    """The tiled LU (include/tlu.h) on the config's matrix: pack + getrf +
    get_u per step, CUDA events on the plan stream; the oracle on the same A bytes (whole matrix
    up to 2e11 flops, else its leading block); e2e through the public API with host buffers."""
    import oracle
    if world > 1:
        if rank == 0:
            print(json.dumps({"method": "lu", "unavailable": "the tiled LU runs on one GPU (replicas only)"}))
        return 0
    m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
    threads = len(os.sched_getaffinity(0))
    A_host = np.asfortranarray(tqr_inputs.make(m, n, cfg["dist"], cfg["seed"]))
    flops = oracle.lu_flops_standard(m, n)
    if args.impl == "reference":
        S = A_host if flops <= LU_FULL_ORACLE_MAX_FLOPS else np.asfortranarray(
            A_host[:min(m, 6144 // b * b), :min(n, 6144 // b * b)])
        vals = []
        for it in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            oracle.lu_getrf_tiles(S, b, s, nthreads=threads)
            dt = time.perf_counter() - t0
            if it >= args.warmup:
                vals.append(oracle.lu_flops_standard(*S.shape) / dt / 1e9)
        v = statistics.median(vals)
        desc = f"oracle_lu_getrf_tiles on {S.shape[0]}x{S.shape[1]} (leading block of the workload), {threads} threads"
        print(json.dumps({"impl": "reference", "method": "lu", "metric": LU_METRIC, "value": v, "unit": "GFLOP/s",
                          "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": cfg["name"].replace(" QR ", " LU "), "sample": desc},
                          "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
                                           "sample": desc},
                          "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return 0
    import torch
    from paper_0707_3548_b200 import tlu
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    plan = tlu.LUPlan(m, n, b, s, device=local, stream=stream)
    A_pin = torch.from_numpy(np.ascontiguousarray(A_host.T)).pin_memory()
    dev = f"cuda:{local}"
    with torch.cuda.stream(stream):
        A_dev = A_pin.to(dev, non_blocking=True)
        At, W, piv = plan.alloc()
        U = torch.zeros((n, min(m, n)), dtype=torch.float64, device=dev)
    stream.synchronize()
    for _ in range(args.warmup):
        plan.pack(A_dev, At)
        plan.getrf(At, W, piv)
        plan.get_u(At, U)
    stream.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        e0.record(stream)
        for kk in range(args.steps):
            plan.pack(A_dev, At)
            ev[kk][0].record(stream)
            plan.getrf(At, W, piv)
            ev[kk][1].record(stream)
            plan.get_u(At, U)
        e1.record(stream)
        stream.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    kern_ms = statistics.mean(a.elapsed_time(b_) for a, b_ in ev)
    value = flops / (ms * 1e-3) / 1e9
    U_g = U.cpu().numpy().T
    piv_g = piv.cpu().numpy()
    # e2e: host A in (pinned), pack, getrf, get_u, U out -- every step, serial on the plan stream
    e2e = None
    if not args.no_e2e:
        U_pin = torch.empty((n, min(m, n)), dtype=torch.float64).pin_memory()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                A_dev.copy_(A_pin, non_blocking=True)
            plan.pack(A_dev, At)
            plan.getrf(At, W, piv)
            plan.get_u(At, U)
            with torch.cuda.stream(stream):
                U_pin.copy_(U, non_blocking=True)
        f1.record(stream)
        stream.synchronize()
        ems = f0.elapsed_time(f1) / args.steps
        e2e = {"value": flops / (ems * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ems,
               "h2d_bytes_per_step": m * n * 8, "d2h_bytes_per_step": n * min(m, n) * 8,
               "note": "A in from pinned host memory, U out, every step, serial on the plan stream"}
    cpu, parity = None, None
    if not args.no_cpu_baseline:
        full = flops <= LU_FULL_ORACLE_MAX_FLOPS
        S = A_host if full else np.asfortranarray(A_host[:min(m, 6144 // b * b), :min(n, 6144 // b * b)])
        t0 = time.perf_counter()
        At_o, _, piv_o = oracle.lu_getrf_tiles(S, b, s, nthreads=threads)
        dt = time.perf_counter() - t0
        desc = (f"oracle_lu_getrf_tiles on {'the full' if full else 'the leading'} {S.shape[0]}x{S.shape[1]} "
                f"{'workload (the same A bytes)' if full else 'block of the workload matrix (same bytes)'}, "
                f"b={b} s={s}, {threads} threads")
        cpu = {"value": oracle.lu_flops_standard(*S.shape) / dt / 1e9, "unit": "GFLOP/s", "cores": threads,
               "kind": "oracle", "sample": desc, "seconds": dt, "same_config": full}
        if full:
            U_o = oracle.get_r(At_o, m, n, b)
            rho = max(1.0, float(np.max(np.abs(U_o)) / np.max(np.abs(A_host))))
            tol = 1e-10 * float(np.linalg.norm(A_host)) * rho
            same = bool(np.array_equal(piv_g, piv_o))
            parity = {"pivots_equal": same, "growth_rho": rho,
                      "what": "GPU factors of the last timed step vs the oracle on the same A (DESIGN.md LU10)"}
            if same:
                err = float(np.max(np.abs(U_g - U_o)))
                parity.update({"U_max_abs_diff_vs_oracle": err, "tol": tol, "ok": err <= tol})
            else:
                # pivots decided by rounding (the oracle itself moves thousands of pivots under a
                # one-ulp perturbation of A here): check what is unique (LU10)
                parity.update(lu_property_parity(At.cpu().numpy(), W.cpu().numpy(), piv_g, U_g, A_host, b, s,
                                                 threads, None))
        else:
            # the oracle cannot factor the whole matrix within the bench's budget: the GPU's
            # factors are checked for what is unique, the transformation on sampled tile columns
            qq = -(-n // b)
            parity = {"what": "valid pairwise-pivoting elimination: |multipliers| <= 1 and the recorded "
                              "transformation (replayed by the oracle from the GPU's factors) maps tile columns "
                              f"0 and {qq - 1} of A to U (DESIGN.md LU10)"}
            parity.update(lu_property_parity(At.cpu().numpy(), W.cpu().numpy(), piv_g, U_g, A_host, b, s, threads,
                                             [0, qq - 1]))
    achieved = flops / (kern_ms * 1e-3) / 1e12
    try:  # one ncu --set full capture of the LU executor on this workload (profiles/traffic.json)
        lu_traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get("LU_" + args.config)
    except (OSError, ValueError):
        lu_traffic = None
    line = {"metric": LU_METRIC, "method": "lu", "value": value, "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"].replace(" QR ", " LU "), "m": m, "n": n, "b": b, "s": s,
                       "dist": cfg["dist"], "seed": cfg["seed"], "parallelism": "1 GPU",
                       "l2": (f"inputs {m * n * 8 / 2**30:.1f} GiB > 126 MB L2; no flush between steps"
                              if m * n * 8 > (1 << 28) else "inputs smaller than L2 (not flushed)"),
                       "step": "pack + getrf (persistent DAG executor, pairwise pivoting) + get_u"},
            "pct_of_fp64_peak": 100.0 * value / (FP64_PEAK_TFLOPS * 1e3),
            "executed_gflops": tlu.flops_tiled(m, n, b, s) / (ms * 1e-3) / 1e9,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS, "traffic": lu_traffic and lu_traffic["bytes"],
                         "traffic_source": lu_traffic and (f"dram__bytes_read.sum + dram__bytes_write.sum per "
                                                           f"launch, {lu_traffic['source']}"),
                         "kernel": f"lu_exec_kernel<{b},{s}> (tlu_getrf)", "kernel_ms": kern_ms,
                         "flops_per_launch": flops,
                         "peak_source": "fp64 DMMA.8x8x4 measured 37.14 TFLOP/s (profiles/r01_m0_fp64_probe.txt)"},
            "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
            "gpu_launches": 3 * args.steps,   # pack, executor, get_u (+ a cudaMemsetAsync of the counters)
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    cfg = dict(tqr_inputs.CONFIGS[args.config])
    cfg["name"] = {"C1": "C1 square QR m=n=256 b=64 s=16 U[-0.5,0.5)",
                   "C2": "C2 square QR m=n=4096 b=128 s=32 U[-0.5,0.5)",
                   "C3": "C3 square QR m=n=16384 b=256 s=32 U[-0.5,0.5)",
                   "C4": "C4 tall-skinny QR m=131072 n=2048 b=256 s=32 N(0,1)",
                   "C5": "C5 square QR m=n=65536 b=512 s=64 U[-0.5,0.5)"}[args.config]
    if args.method == "lu":
        return run_lu(args, cfg, rank, world, local)
    if args.impl == "reference":
        return run_reference(args, cfg, rank)

    import torch
    import torch.distributed as dist
    import paper_0707_3548_b200 as tqr
    from paper_0707_3548_b200 import dist as tdist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
    G = world if world > 1 else args.emulate_ranks
    stream = torch.cuda.Stream()
    tall = args.tiles == "2bxb"
    plan = tqr.Plan(m, n, b, s, device=local, stream=stream, nranks=G, rank=rank if world > 1 else 0,
                    emulate=world == 1 and G > 1, tall=tall, locality=args.schedule == "locality")
    if world > 1:
        tdist.connect(plan)   # one-time CUDA IPC blob exchange
    A_host = tqr_inputs.make(m, n, cfg["dist"], cfg["seed"])                  # one matrix, every rank
    A_pin = torch.from_numpy(np.ascontiguousarray(A_host.T)).pin_memory()     # column-major storage, pinned
    del A_host
    # this rank's tile columns of A (column-major storage rows = matrix columns)
    my_tiles = tdist.owned_columns(plan.q, G, rank) if world > 1 else list(range(plan.q))
    my_cols = [(j * b, min(n, (j + 1) * b)) for j in my_tiles]
    with torch.cuda.stream(stream):
        A_dev = A_pin.to(f"cuda:{local}", non_blocking=True)
        At, T = plan.alloc()
        R = torch.zeros((n, min(m, n)), dtype=torch.float64, device=f"cuda:{local}")
    stream.synchronize()

    def step():
        plan.pack(A_dev, At)
        plan.geqrf(At, T)
        plan.get_r(At, R)

    flops = tqr.flops_standard(m, n)
    # executed count at the executor's internal inner block (b = 512, s = 64 runs SI = 16 blocks,
    # DESIGN.md R16; the off-diagonal T blocks of form_t are not counted)
    flops_exec = tqr.flops_tiled(m, n, b, plan.info()["inner"])
    for _ in range(args.warmup):
        step()
    stream.synchronize()

    # ---- timed region: K steps, per-step events around the executor launch too ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        e0.record(stream)
        for kk in range(args.steps):
            plan.pack(A_dev, At)
            ev[kk][0].record(stream)
            plan.geqrf(At, T)
            ev[kk][1].record(stream)
            plan.get_r(At, R)
        e1.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    kern_ms = statistics.mean(a.elapsed_time(b_) for a, b_ in ev)
    if world > 1:
        t = torch.tensor([ms, kern_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_ms = t.tolist()
    value = flops / (ms * 1e-3) / 1e9     # one matrix for the whole job (strong scaling)

    # ---- e2e: host buffers through the public API.  Every step copies its own input in
    #      (H2D of this rank's columns of A from pinned memory), packs, factors, extracts R
    #      and copies its own result out (D2H of this rank's columns of R).  The copies run on
    #      a second stream with double-buffered device A and R, so step s+1's H2D and step
    #      s-1's D2H overlap step s's factorization (a serving pipeline). ----
    e2e = None
    if not args.no_e2e:
        dev = f"cuda:{local}"
        free_b, _ = torch.cuda.mem_get_info(dev)
        dbl = free_b > 1.15 * (A_dev.numel() + R.numel()) * 8   # room for the second buffers?
        A_bufs = [A_dev, torch.empty_like(A_dev) if dbl else A_dev]
        R_bufs = [R, torch.zeros_like(R) if dbl else R]
        R_pins = [torch.empty((n, min(m, n)), dtype=torch.float64).pin_memory() for _ in range(2)]
        cst = torch.cuda.Stream(device=dev)   # H2D
        dst = torch.cuda.Stream(device=dev)   # D2H
        ev = {key: [torch.cuda.Event() for _ in range(2)] for key in ("h2d", "packed", "r", "d2h")}
        issued = {key: [False, False] for key in ev}

        def e2e_run(nsteps):
            for st_ in range(nsteps):
                bf = st_ % 2
                with torch.cuda.stream(cst):   # H2D of this step's A once its buffer is free
                    if issued["packed"][bf]:
                        cst.wait_event(ev["packed"][bf])
                    for c0, c1 in my_cols:
                        A_bufs[bf][c0:c1].copy_(A_pin[c0:c1], non_blocking=True)
                    ev["h2d"][bf].record(cst); issued["h2d"][bf] = True
                stream.wait_event(ev["h2d"][bf])
                plan.pack(A_bufs[bf], At)
                ev["packed"][bf].record(stream); issued["packed"][bf] = True
                plan.geqrf(At, T)
                if issued["d2h"][bf]:
                    stream.wait_event(ev["d2h"][bf])   # R buffer read out by step s-2
                plan.get_r(At, R_bufs[bf])
                ev["r"][bf].record(stream); issued["r"][bf] = True
                with torch.cuda.stream(dst):   # D2H of this step's R
                    dst.wait_event(ev["r"][bf])
                    for c0, c1 in my_cols:
                        R_pins[bf][c0:c1].copy_(R_bufs[bf][c0:c1], non_blocking=True)
                    ev["d2h"][bf].record(dst); issued["d2h"][bf] = True

        e2e_run(2)
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(cst)
        e2e_run(args.steps)
        f1.record(dst)       # after the last D2H (D2H stream order)
        torch.cuda.synchronize()
        barrier()
        ems = f0.elapsed_time(f1) / args.steps
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        del A_bufs[1], R_bufs[1]
        e2e = {"value": flops / (ems * 1e-3) / 1e9, "unit": "GFLOP/s", "double_buffered": dbl,
               "h2d_bytes_per_step": sum(c1 - c0 for c0, c1 in my_cols) * m * 8,
               "d2h_bytes_per_step": sum(c1 - c0 for c0, c1 in my_cols) * min(m, n) * 8,
               "ms_per_step": ems,
               "note": "per rank: its own tile columns of A in, of R out, every step; H2D and D2H on their "
                       "own streams, double-buffered, overlapping the neighbouring steps' factorization"}

    # ---- form Q explicitly (tqr_orgqr), once, after the timed region ----
    form_q = None
    if world == 1 and not args.no_e2e and not tall:
        qb = -(-n // b)
        free_b, _ = torch.cuda.mem_get_info(f"cuda:{local}")
        if free_b > 1.2 * plan.p * qb * b * b * 8:
            Qt = torch.empty(plan.p * qb * b * b, dtype=torch.float64, device=f"cuda:{local}")
            plan.orgqr(At, T, n, Qt)      # warm-up (builds the apply-Q schedule)
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record(stream)
            plan.orgqr(At, T, n, Qt)
            q1.record(stream)
            stream.synchronize()
            qms = q0.elapsed_time(q1)
            k_ = min(m, n)
            qfl = 4.0 * m * n * k_ - 2.0 * (m + n) * k_ * k_ + 4.0 / 3.0 * k_ ** 3   # DORGQR count
            form_q = {"ms": qms, "gflops": qfl / (qms * 1e-3) / 1e9, "flop_model": "4mnk-2(m+n)k^2+4k^3/3, k=n",
                      "pct_of_fp64_peak": 100.0 * qfl / (qms * 1e-3) / (FP64_PEAK_TFLOPS * 1e12)}
            del Qt

    # ---- optional trace of one extra step ----
    if args.trace and rank == 0 and world == 1:
        tplan = tqr.Plan(m, n, b, s, device=local, stream=stream, trace=True, nranks=G, emulate=G > 1, tall=tall)
        tplan.pack(A_dev, At)
        tplan.geqrf(At, T)
        tplan.sync()
        rec = tplan.trace()
        t0 = int(rec[:, 6].min())
        with open(args.trace, "w") as f:
            json.dump({"fields": ["kind", "k", "i", "j", "slice", "sm", "start_ns", "end_ns"],
                       "t0": t0, "records": rec.tolist()}, f)
        tplan.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    cpu, parity = None, None
    if not args.no_cpu_baseline and world == 1:
        # The oracle as it stands on the host cores.  Up to C4 it factors the WHOLE workload
        # (the same A bytes the GPU factored) and the GPU's R of the last timed step is
        # compared with it elementwise (BJ north_star: within 1e-10 * ||A||_F); C5 (3.8e14
        # flops, hours on the host) times the oracle on a leading-block sample instead.
        threads = len(os.sched_getaffinity(0))
        A_host = A_pin.numpy().T                          # m x n, Fortran order (no copy)
        if flops <= FULL_ORACLE_MAX_FLOPS:
            import oracle
            v, dt, At_o, _ = time_oracle(A_host, cfg, threads, h=2 if tall else 1)
            desc = (f"oracle_geqrf_tiles on the full {m}x{n} workload (the same A bytes), b={b} s={s}"
                    f"{', 2b x b tiles' if tall else ''}, {threads} threads, one factorization")
            R_o = oracle.get_r(At_o, m, n, b)
            del At_o
            R_g = R.cpu().numpy().T
            nA = float(np.linalg.norm(A_host))
            err = float(np.max(np.abs(R_g - R_o)))
            parity = {"R_max_abs_diff_vs_oracle": err, "tol": 1e-10 * nA, "ok": err <= 1e-10 * nA,
                      "what": "GPU R of the last timed step vs the oracle's R on the same A, elementwise"}
            del R_o, R_g
            cpu = {"value": v, "unit": "GFLOP/s", "cores": threads, "kind": "oracle", "sample": desc, "seconds": dt,
                   "same_config": True}
        else:
            S = sample_block(cfg, A_host)
            v, dt, _, _ = time_oracle(S, cfg, threads)
            desc = (f"oracle_geqrf_tiles on the leading {S.shape[0]}x{S.shape[1]} block of the workload matrix "
                    f"(same bytes), b={b} s={s}, {threads} threads, one factorization")
            cpu = {"value": v, "unit": "GFLOP/s", "cores": threads, "kind": "oracle", "sample": desc, "seconds": dt,
                   "same_config": False}

    achieved = flops / world / (kern_ms * 1e-3) / 1e12   # this GPU's share of the job, per launch
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config)
        if tr and world == 1:
            traffic = {"bytes": tr["bytes"], "source": tr["source"],
                       "flop_per_dram_byte": flops / tr["bytes"]}
    except (OSError, ValueError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "m": m, "n": n, "b": b, "s": s, "dist": cfg["dist"],
                   "seed": cfg["seed"],
                   "parallelism": (f"1D block-cyclic tile columns over {world} GPUs, V/T by NVLink peer stores"
                                   if world > 1 else ("1 GPU" if G == 1 else f"1 GPU, {G} emulated ranks")),
                   "l2": (f"inputs {m * n * 8 / 2**30:.1f} GiB > 126 MB L2; no flush between steps"
                          if m * n * 8 > (1 << 28) else "inputs smaller than L2 (not flushed)"),
                   "step": "pack + geqrf (persistent DAG executor) + get_r",
                   "tiles": "2b x b (TQR_FLAG_TALL_TILES)" if tall else "b x b",
                   "schedule": "locality (TQR_FLAG_LOCALITY)" if args.schedule == "locality" else "critical path"},
        "pct_of_fp64_peak": 100.0 * value / (world * FP64_PEAK_TFLOPS * 1e3),
        "executed_gflops": flops_exec / (ms * 1e-3) / 1e9,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic and traffic["bytes"],
                     "traffic_source": traffic and (f"dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                                                    f"{traffic['source']} ({traffic['flop_per_dram_byte']:.1f} "
                                                    f"flop per DRAM byte)"),
                     "kernel": f"exec_kernel<{b},{s},mode 0> (tqr_geqrf)", "kernel_ms": kern_ms,
                     "flops_per_launch": flops / world,
                     "peak_source": "fp64 DMMA.8x8x4 measured 37.14 TFLOP/s (profiles/r01_m0_fp64_probe.txt); "
                                    "MEASURED_PEAKS.json has no fp64 entry"},
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        "form_q": form_q,
        # pack, [rank barrier,] executor, [form_t: b*s > 8192, the executor's internal blocks
        # are narrower than s], get_r
        "gpu_launches": (3 + (world > 1) + (b * s > 8192)) * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
