#!/usr/bin/env python
"""bench.py — CGGM Newton-iteration evaluations/s at p=40k, q=20k (BASELINE.json `large`).

One step = one Newton-iteration evaluation at (Lambda*, Theta*):
  cggm_invert_logdet(Lambda)  -> Sigma, log|Lambda|, PD            (potrf + trtri + lauum)
  cggm_psi_grad(+fused active sets) -> Psi, grad_Lambda, grad_Theta, S_Lambda, S_Theta, ||grad^S||_1
  cggm_objective(Lambda_trial = Lambda, Theta) with its own fresh Cholesky (a line-search trial)
S_yy (per-dataset setup) is computed once before the timed region and reported separately.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cggm|reference] [--config large]

N > 1 (torchrun): the n samples are sharded over the ranks; rank 0 inverts Lambda and broadcasts
Sigma; Psi and grad_Theta partials are all-reduced over NCCL (strong scaling: one evaluation of
the fixed `large` problem per step).  `--impl reference` times the CPU oracle (oracle/, numpy
fp64) on a bounded sample of the same workload, on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CGGM Newton-iteration evals/s at p=40k,q=20k; FP64 tensor/HBM % of peak"
UNIT = "evals/s"


def alg_flops(n, p, q, nnz_theta):
    """Algorithmic FP64 flops of one evaluation: (4/3) q^3 (potrf x2 + trtri +
    lauum) + 2nq^2 (R = W Sigma) + nq^2 (Psi, symmetric) + 2npq (grad_Theta) + nq^2 (trsm) +
    2 n nnz(Theta) (SpMM).  S_xx, dense X Theta and (X^T W) Sigma are avoided and not counted."""
    gemm = (4.0 / 3.0) * q ** 3 + 4.0 * n * q * q + 2.0 * n * p * q
    return gemm, gemm + 2.0 * n * nnz_theta


def phase_flops(n, p, q):
    return {"chol_gemm": q ** 3, "lauum": q ** 3 / 3.0, "w_sigma": 2.0 * n * q * q, "psi_gradL": 1.0 * n * q * q,
            "grad_theta": 2.0 * n * p * q, "obj_trsm": 1.0 * n * q * q}


GEMM_TAGS = ("chol_gemm", "lauum", "w_sigma", "psi_gradL", "grad_theta", "obj_trsm")


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0   # B200_PROFILING.md fallback


HBM_PEAK_GBS = _hbm_peak()


def _dominant_traffic():
    """dram read+write bytes per launch of the largest GEMM launch (X^T E since Sigma is assembled inside
    the recursion), from the committed ncu --set full capture (profiles/r02_ncu_dominant.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_ncu_dominant.json")))
        return d["dram_read_bytes"] + d["dram_write_bytes"]
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            try:
                pw.append(float(parts[3]))
            except ValueError:
                pass
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [s for s in sm if mx is None or s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_median": statistics.median(pw) if pw else None}


def run_env():
    """GPU / driver / CUDA / host description for the JSON line (SURVEY.md §8(d) timing protocol)."""
    import torch
    env = {"gpu": torch.cuda.get_device_name(0), "torch": torch.__version__, "cuda_runtime": torch.version.cuda}
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=driver_version", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=20).stdout.strip().splitlines()
        env["driver"] = out[0] if out else None
    except (OSError, subprocess.TimeoutExpired):
        env["driver"] = None
    try:
        with open("/proc/cpuinfo") as f:
            env["cpu_model"] = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        env["cpu_model"] = None
    env["host_cores"] = os.cpu_count()
    return env


# ----------------------------------------------------------------------------- oracle (CPU) leg
def oracle_sample(P, qs, ps):
    """Bounded sample of the `large` workload for the CPU oracle: the leading qs outputs, ps
    inputs and all n samples (Lambda*, Theta* restricted to that block)."""
    from synth.cggm_inputs import Csc
    lam = P.lam_star
    d = lam.to_scipy()[:qs, :qs].tocsc()
    d.sort_indices()
    lam_s = Csc(qs, qs, d.indptr.astype(np.int64), d.indices.astype(np.int32), d.data.copy())
    t = P.theta_star.to_scipy()[:ps, :qs].tocsc()
    t.sort_indices()
    th_s = Csc(ps, qs, t.indptr.astype(np.int64), t.indices.astype(np.int32), t.data.copy())
    X = np.asfortranarray(P.X[:, :ps])
    Y = np.asfortranarray(P.Y[:, :qs])
    return X, Y, lam_s, th_s


def oracle_eval_seconds(X, Y, lam, th, lam_L, lam_T):
    from oracle import cggm_oracle as O
    t0 = time.perf_counter()
    Syy, _ = O.covariances(X, Y)    # setup, excluded below
    t1 = time.perf_counter()
    Sig, ld, ok, fc = O.invert_logdet(lam.to_dense())
    r = O.psi_grad(X, Y, th, Sig, Syy, None)
    O.active_set(r["GradL"], r["GradT"], lam, th, lam_L, lam_T)
    O.min_norm_subgradient(r["GradL"], r["GradT"], lam, th, lam_L, lam_T)
    O.objective(X, Y, lam, th, lam_L, lam_T)
    t2 = time.perf_counter()
    return t2 - t1, t1 - t0


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = [d.get("num_threads", 1) for d in info if d.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(P, qs=5000, ps=10000):
    X, Y, lam_s, th_s = oracle_sample(P, qs, ps)
    secs, _ = oracle_eval_seconds(X, Y, lam_s, th_s, P.lam_L, P.lam_T)
    _, full = alg_flops(P.n, P.p, P.q, P.theta_star.nnz)
    _, samp = alg_flops(P.n, ps, qs, th_s.nnz)
    est = secs * full / samp
    out = {"value": 1.0 / est, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
           "sample": f"one oracle evaluation on the leading {qs} outputs x {ps} inputs x all {P.n} samples of "
                     f"`large` ({secs:.2f} s), extrapolated by algorithmic flops x{full / samp:.0f}",
           "sample_seconds": secs}
    try:   # the same oracle on one core (one thread and all cores), a smaller block
        from threadpoolctl import threadpool_limits
        q1, p1 = 1500, 3000
        X1, Y1, lam1, th1 = oracle_sample(P, q1, p1)
        with threadpool_limits(limits=1):
            s1, _ = oracle_eval_seconds(X1, Y1, lam1, th1, P.lam_L, P.lam_T)
        _, samp1 = alg_flops(P.n, p1, q1, th1.nnz)
        out["single_thread"] = {"value": samp1 / full / s1, "unit": UNIT, "cores": 1, "sample_seconds": s1,
                                "sample": f"leading {q1} outputs x {p1} inputs x all {P.n} samples, "
                                          f"extrapolated x{full / samp1:.0f}"}
    except ImportError:
        pass
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth.cggm_inputs import make_problem
    P = make_problem(args.config)
    qs, ps = 3000, 6000
    X, Y, lam_s, th_s = oracle_sample(P, qs, ps)
    _, full = alg_flops(P.n, P.p, P.q, P.theta_star.nnz)
    _, samp = alg_flops(P.n, ps, qs, th_s.nnz)
    for _ in range(args.warmup):
        oracle_eval_seconds(X, Y, lam_s, th_s, P.lam_L, P.lam_T)
    times = [oracle_eval_seconds(X, Y, lam_s, th_s, P.lam_L, P.lam_T)[0] for _ in range(args.steps)]
    est = sum(times) / len(times) * full / samp
    value = 1.0 / est
    cb = {"value": value, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
          "sample": f"per step: one oracle evaluation on the leading {qs} outputs x {ps} inputs x all {P.n} samples "
                    f"of `{args.config}`, extrapolated by algorithmic flops x{full / samp:.0f}"}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n": P.n, "p": P.p, "q": P.q},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- FP32 variant
def _bf16_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        return 1628.6   # B200_PROFILING.md fallback


def fp32_variant(configs, steps, P_large=None):
    """The FP32 variant (reading A18; north_star "with an FP32 variant", `medium fp64+fp32`): one
    Newton-iteration evaluation in a CGGM_F32 context (3xTF32 on the tcgen05 tensor cores), timed like
    region A at each config.  Roofline: algorithmic flops (the same count as FP64) / step / the 3xTF32
    peak = MEASURED_PEAKS bf16 x 1/2 (the guide's nominal tf32 : bf16 ratio) / 3 products."""
    import torch
    from paper_1509_04681_b200 import Context, DeviceCsc, newton_evaluation, to_device_colmajor
    from synth.cggm_inputs import make_problem
    peak = _bf16_peak() * 0.5 / 3.0
    out = {"engine": "3xTF32 tcgen05.mma.kind::tf32 (hi/lo split, TMEM accumulators, chunked fp32 drain)",
           "peak_tflops_3xtf32": peak, "peak_source": "MEASURED_PEAKS.json bf16_tflops x 0.5 (tf32 : bf16) / 3"}
    for name in configs:
        P = P_large if (name == "large" and P_large is not None) else make_problem(name)
        _, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
        ctx = Context(0, dtype="f32")
        f32 = torch.float32
        X, Y = to_device_colmajor(P.X, dtype=f32), to_device_colmajor(P.Y, dtype=f32)
        L, T = DeviceCsc.from_host(lam, dtype=f32), DeviceCsc.from_host(th, dtype=f32)
        Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
        bufs = {k: torch.empty(0, dtype=torch.int32, device="cuda") for k in ("L_row", "L_col", "T_row", "T_col")}
        try:
            newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
        except Exception as exc:
            if getattr(exc, "status", None) != 6:
                raise
        mL, mT = ctx.last_active_sizes
        for k, c_ in (("L_row", mL), ("L_col", mL), ("T_row", mT), ("T_col", mT)):
            bufs[k] = torch.empty(int(c_ * 1.1) + 1024, dtype=torch.int32, device="cuda")
        for _ in range(3):
            r = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            r = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, bufs)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        _, fl = alg_flops(P.n, P.p, P.q, P.theta_star.nnz)
        ach = fl / (ms * 1e-3) / 1e12
        out[name] = {"value": 1e3 / ms, "unit": UNIT, "ms_per_step": ms, "steps": steps, "dtype": "f32",
                     "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                                  "frac": ach / peak},
                     "f": r["objective"]["f"], "m_L": r["active"]["m_L"], "m_T": r["active"]["m_T"]}
        del ctx, X, Y, L, T, Syy, bufs, r
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- launch
def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def maybe_self_launch(args):
    """`python bench.py --gpus N` without torchrun: re-launch as N ranks through
    torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous).  Under torchrun, WORLD_SIZE
    must equal --gpus."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None:
        if args.gpus > 1 and args.impl == "cggm":
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
                   *sys.argv[1:]]
            sys.exit(subprocess.call(cmd))
        return
    if int(env_world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")


def l2_note(P):
    q2, pq = 8.0 * P.q * P.q, 8.0 * P.p * P.q
    return (f"inputs larger than L2 (126 MB): Sigma/Psi/grad_Lambda {q2 / 1e9:.1f} GB each, "
            f"grad_Theta {pq / 1e9:.1f} GB, X {8.0 * P.n * P.p / 1e9:.2f} GB")


def gather_objects(obj, world):
    import torch.distributed as dist
    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


# ----------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cggm", choices=["cggm", "reference"])
    ap.add_argument("--config", default="large")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--allreduce", default="nccl", choices=["nccl", "peer"],
                    help="N > 1: Psi / grad_Theta partials summed by NCCL or over CUDA IPC peer memory")
    ap.add_argument("--inverse", default="auto", choices=["auto", "rank0", "distributed"],
                    help="N > 1: Sigma on rank 0 + broadcast, or the block-cyclic distributed inverse "
                         "(NEXT-3); auto = distributed from 3 GPUs")
    ap.add_argument("--grad-theta", default="reduce_scatter", choices=["reduce_scatter", "allreduce"],
                    help="N > 1: grad_Theta by reduce-scattered column ranges with compact-list all-gather "
                         "(no p x q buffer), or the full p x q all-reduce")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the FP32-variant timings (medium, large)")
    ap.add_argument("--no-variants", action="store_true", help="skip the eager / changing-Lambda step timings")
    ap.add_argument("--peak-seconds", type=float, default=2.0)
    ap.add_argument("--stream-grad-theta", action="store_true",
                    help="do not store the p x q grad_Theta (streamed into the active sets); default for `sharded`")
    args = ap.parse_args()
    if args.config == "sharded":
        args.stream_grad_theta = True
    maybe_self_launch(args)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # (CGGM_BENCH_DEVICE / CGGM_BENCH_BACKEND: functional check of the multi-rank path on a one-GPU
    # box -- every rank on one device over gloo; such a run's numbers are not measurements)
    functional = "CGGM_BENCH_DEVICE" in os.environ
    local = int(os.environ.get("CGGM_BENCH_DEVICE", local))
    if not functional and world > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    backend = os.environ.get("CGGM_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator rank / nranks in the log
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        print(f"[bench] rank {dist.get_rank()} of world {dist.get_world_size()} on cuda:{local} "
              f"({backend})", file=sys.stderr, flush=True)

    from paper_1509_04681_b200 import Context, DeviceCsc, colmajor_empty
    from paper_1509_04681_b200.sharded import CudaBackend, ShardedEvaluator, shard_rows
    from paper_1509_04681_b200 import _abi
    from synth.cggm_inputs import make_problem

    t_gen = time.perf_counter()
    P = make_problem(args.config)
    t_gen = time.perf_counter() - t_gen
    a, b = shard_rows(P.n, world, rank)
    n_loc = b - a
    label, lam_h, th_h = [pt for pt in P.points if pt[0] == "truth"][0]

    def to_dev(A):
        t = colmajor_empty(A.shape[0], A.shape[1])
        t.copy_(torch.from_numpy(np.asfortranarray(A)))
        return t

    X = to_dev(P.X[a:b])
    Y = to_dev(P.Y[a:b])
    Lam = DeviceCsc.from_host(lam_h)
    Th = DeviceCsc.from_host(th_h)
    ctx = Context(local, validate=1)
    stream = torch.cuda.current_stream()

    # FP64 tensor-pipe peak, measured live (MEASURED_PEAKS.json has no FP64 entry)
    tf, ms = ctypes.c_double(), ctypes.c_double()
    ctx._check(ctx.lib.cggm_test_fp64_peak(ctx.h, args.peak_seconds, ctypes.byref(tf), ctypes.byref(ms)))
    peak_tflops = tf.value
    # L2 -> SM read bandwidth, measured live (the SpMM gathers from L2: its roofline denominator)
    l2g, l2ms = ctypes.c_double(), ctypes.c_double()
    ctx._check(ctx.lib.cggm_test_l2_peak(ctx.h, 1.0, ctypes.byref(l2g), ctypes.byref(l2ms)))
    l2_peak_gbs = l2g.value

    dist_inv = args.inverse == "distributed" or (args.inverse == "auto" and world >= 3)
    ev = ShardedEvaluator(CudaBackend(ctx), distributed_inverse=dist_inv, split_objective=not dist_inv,
                          peer_allreduce=args.allreduce == "peer", grad_theta=args.grad_theta)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    Syy = ev.setup(X, Y, P.n)
    e1.record(stream)
    torch.cuda.synchronize()
    setup_ms = e0.elapsed_time(e1)

    q, p = P.q, P.p
    if world == 1:
        # single GPU: fused active sets in the Psi/grad call, preallocated outputs
        bufs = {"Sigma": colmajor_empty(q, q), "Psi": colmajor_empty(q, q), "GradL": colmajor_empty(q, q)}
        if not args.stream_grad_theta:
            bufs["GradT"] = colmajor_empty(p, q)
        from paper_1509_04681_b200.api import newton_evaluation
        # size the active-set lists with the two-call pattern (capacity 0 -> required sizes)
        for k in ("L_row", "L_col", "T_row", "T_col"):
            bufs[k] = torch.empty(0, dtype=torch.int32, device="cuda")
        try:
            newton_evaluation(ctx, X, Y, Syy, Lam, Th, P.lam_L, P.lam_T, True, bufs,
                              stream_grad_theta=args.stream_grad_theta)
        except Exception as exc:  # CGGM_ERR_CAPACITY carries the sizes
            if getattr(exc, "status", None) != 6:
                raise
        m = ctx.last_active_sizes
        capL, capT = int(m[0] * 1.10) + 1024, int(m[1] * 1.10) + 1024
        for k, cap in (("L_row", capL), ("L_col", capL), ("T_row", capT), ("T_col", capT)):
            bufs[k] = torch.empty(cap, dtype=torch.int32, device="cuda")

        def step():
            return newton_evaluation(ctx, X, Y, Syy, Lam, Th, P.lam_L, P.lam_T, True, bufs,
                                     stream_grad_theta=args.stream_grad_theta)
    else:
        def step():
            return ev.evaluate(X, Y, Lam, Th, P.lam_L, P.lam_T, True)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, k, pre=None):
        """k calls of fn between events on the launching stream, barrier + synchronize on both sides,
        max over ranks (ms for all k)."""
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(k):
            if pre is not None:
                pre(i)
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1))

    for _ in range(max(args.warmup, 0)):
        last = step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    # ---------------- timed region A: the reported value (no library profiling events inside)
    l0 = ctx.launch_count()
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        last = step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    elapsed = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    elapsed = max_over_ranks(elapsed)
    launches_all = gather_objects(launches, world)
    clk_all = gather_objects(clk, world)

    # ---------------- per-step distribution (after region A, which it does not perturb): each step
    # bracketed by its own events, at least 10 steps (median with p10 / p90)
    n_dist = max(10, args.steps)
    ev_pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_dist)]
    for a_, b_ in ev_pairs:
        a_.record(stream)
        step()
        b_.record(stream)
    torch.cuda.synchronize()
    per_step = sorted(a_.elapsed_time(b_) for a_, b_ in ev_pairs)
    q10 = per_step[max(0, int(round(0.1 * (n_dist - 1))))]
    q90 = per_step[min(n_dist - 1, int(round(0.9 * (n_dist - 1))))]
    step_dist = {"n": n_dist, "median_ms": statistics.median(per_step), "p10_ms": q10, "p90_ms": q90,
                 "min_ms": per_step[0], "max_ms": per_step[-1]}
    if world > 1:
        step_dist["median_ms_max_over_ranks"] = max_over_ranks(step_dist["median_ms"])

    # ---------------- step variants (honest timing of the graph replay): the plain stream launches
    # (CGGM_OPT_GRAPHS = 0), and a Lambda whose values change every step (new values written into
    # the same CSC buffers before each evaluation -- the replayed graph reads them; the write is timed)
    variants = None
    if world == 1 and not args.no_variants:
        kv = max(3, min(args.steps, 5))
        ctx.set_option(_abi.CGGM_OPT_GRAPHS, 0)
        step()
        eager_ms = timed(step, kv) / kv
        ctx.set_option(_abi.CGGM_OPT_GRAPHS, 1)
        v0 = Lam.val.clone()
        offd = (Lam.rowidx.long() != torch.repeat_interleave(
            torch.arange(q, device="cuda"), Lam.colptr[1:] - Lam.colptr[:-1])).to(torch.float64)
        scales = [1.0 - 0.002 * (i % 5) for i in range(kv + 2)]
        vals = [v0 * (1.0 - offd * (1.0 - s_)) for s_ in scales]   # off-diagonals scaled: stays PD (chain)

        def pre(i):
            Lam.val.copy_(vals[i % len(vals)])
        for i in range(2):
            pre(i + kv)
            step()
        chg_ms = timed(step, kv, pre=pre) / kv
        Lam.val.copy_(v0)
        last = step()
        torch.cuda.synchronize()
        # the other grad_Theta form: stored (p x q) <-> not stored, S_Theta selected in the X^T E epilogue (K01)
        other = not args.stream_grad_theta

        def step_other():
            return newton_evaluation(ctx, X, Y, Syy, Lam, Th, P.lam_L, P.lam_T, True, bufs, stream_grad_theta=other)
        if other or "GradT" in bufs:
            for _ in range(2):
                step_other()
            other_ms = timed(step_other, kv) / kv
        else:
            other_ms = None
        variants = {"graph_replay_ms": elapsed / args.steps, "eager_ms": eager_ms, "changing_lambda_ms": chg_ms,
                    ("grad_theta_not_stored_ms" if other else "grad_theta_stored_ms"): other_ms,
                    "steps": kv,
                    "changing_lambda": "off-diagonal values of Lambda* scaled by 1, 0.998, ..., 0.992 in turn, "
                                       "written into the same CSC before each step (copy timed); the graph "
                                       "replays on the new values"}

    # ---------------- secondary: the factor-reuse evaluation: the accepted trial's
    # inverse factor seeds the next Sigma (CGGM_OPT_FACTOR_REUSE; here the trial Lambda is the
    # evaluation's Lambda, as for the accepted unit step of a converging line search)
    reuse = None
    if world == 1:
        ctx.set_option(_abi.CGGM_OPT_FACTOR_REUSE, 1)
        for _ in range(2):
            step()
        r_ms = timed(step, args.steps) / args.steps
        ctx.set_option(_abi.CGGM_OPT_FACTOR_REUSE, 0)
        _, r_all = alg_flops(P.n, P.p, P.q, P.theta_star.nnz)
        r_all -= P.q ** 3 / 3.0
        reuse = {"value": 1e3 / r_ms, "unit": UNIT, "ms_per_step": r_ms, "alg_flops_per_step": r_all,
                 "step_frac_of_peak": r_all / (r_ms * 1e-3) / 1e12 / peak_tflops,
                 "what": "Sigma from the previous evaluation's trial inverse (potrf+trtri in the objective, "
                         "lauum for Sigma): (4/3) q^3 -> q^3"}

    # ---------------- timed region B (attribution only): per-launch CUDA events on the launching
    # streams (library profiling), the same evaluation issued as the serialised separate calls so that
    # every kernel's duration is its own (no overlap with the auxiliary stream)
    prof_steps = max(1, min(args.steps, 3))
    phases, prof_elapsed, rank_phases = {}, None, None
    if world == 1:
        from paper_1509_04681_b200.api import newton_evaluation as _ne

        def step_prof():
            if args.stream_grad_theta:   # the separate calls need a stored grad_Theta
                return _ne(ctx, X, Y, Syy, Lam, Th, P.lam_L, P.lam_T, True, bufs, stream_grad_theta=True)
            return _ne(ctx, X, Y, Syy, Lam, Th, P.lam_L, P.lam_T, True, bufs, composite=False)
        torch.cuda.synchronize()
        # without the recursion lookahead: every kernel runs alone on its stream, so the sum of
        # per-launch durations is the GEMM family's own time
        ctx.set_option(_abi.CGGM_OPT_LOOKAHEAD_MIN, 0)
        step_prof()
        torch.cuda.synchronize()
        ctx.profile(True)
        e0.record(stream)
        for _ in range(prof_steps):
            step_prof()
        e1.record(stream)
        torch.cuda.synchronize()
        prof_elapsed = e0.elapsed_time(e1)
        prof = ctx.profile_read()
        ctx.profile(False)
        ctx.set_option(_abi.CGGM_OPT_LOOKAHEAD_MIN, 256)
        ph_flops = phase_flops(P.n, P.p, P.q)
        for tag, (tms, tcnt) in prof.items():
            if tcnt == 0:
                continue
            d = {"ms_per_step": tms / prof_steps, "launches_per_step": tcnt / prof_steps}
            if tag in ph_flops:
                d["tflops"] = ph_flops[tag] / (tms / prof_steps * 1e-3) / 1e12
            phases[tag] = d
    else:
        # per-rank phase times of one evaluation (events between the evaluator's phases)
        ev.timing = True
        barrier()
        step()
        pt = ev.phase_times()
        ev.timing = False
        rank_phases = gather_objects(pt, world)

    ms_step = elapsed / args.steps
    value = args.steps / (elapsed / 1e3)
    gemm_flops, all_flops = alg_flops(P.n, P.p, P.q, P.theta_star.nnz)
    q_, p_, n_ = P.q, P.p, P.n

    # collectives per evaluation at N > 1 (bytes each rank contributes; achieved = bytes / phase time)
    comm = None
    if world > 1:
        by = {"bcast_sigma": 8.0 * q_ * q_, "allreduce_psi": 8.0 * q_ * q_, "allreduce_grad_theta": 8.0 * p_ * q_,
              "reduce_scatter_grad_theta": 8.0 * p_ * q_}
        comm = {"backend": backend, "allreduce": args.allreduce, "grad_theta": args.grad_theta, "per_rank": []}
        for r_, ph in enumerate(rank_phases):
            d = {"rank": r_, "phase_ms": ph}
            for k_, b_ in by.items():
                if k_ in ph and ph[k_] > 0:
                    alg = b_ / (ph[k_] * 1e-3) / 1e9
                    bus = alg * (2.0 * (world - 1) / world if k_.startswith("allreduce") else
                                 (world - 1) / world if k_.startswith("reduce_scatter") else 1.0)
                    d[k_ + "_GBps"] = {"bytes": b_, "algbw": alg, "busbw": bus}
            comm["per_rank"].append(d)

    # HBM-bound phases: algorithmic bytes per step / the phase's measured time per
    # step in pass B (every launch of the phase bracketed by its own CUDA events)
    hbm = {}
    if world == 1:
        m_L, m_T = last["active"]["m_L"], last["active"]["m_T"]
        spmm_calls = phases.get("spmm", {}).get("launches_per_step", 1.0)
        hbm_alg = {
            # one read of grad_Lambda's upper triangle and of grad_Theta (stored, or its streamed column
            # chunks), 8 bytes written per active entry
            "active_set": 8.0 * (q_ * (q_ + 1) / 2 + p_ * q_) + 8.0 * (m_L + m_T),
            "grad_lambda": 32.0 * q_ * q_,                       # read S_yy, Sigma, Psi, write grad_Lambda
            "spmm": 8.0 * n_ * (p_ + q_) * spmm_calls,           # per call: read X once, write W
        }
        for tag, by_ in hbm_alg.items():
            if tag in phases:
                ms_s = phases[tag]["ms_per_step"]
                gbs = by_ / (ms_s * 1e-3) / 1e9
                hbm[tag] = {"alg_bytes_per_step": by_, "ms_per_step": ms_s, "achieved_gbs": gbs,
                            "frac_of_measured_copy": gbs / HBM_PEAK_GBS}
        if "spmm" in hbm:
            # W = X Theta gathers n values of X per stored Theta entry (X is read from DRAM once and
            # then re-read from L2): bound by L2 -> SM bandwidth, measured live beside it
            l2_by = 8.0 * n_ * P.theta_star.nnz * spmm_calls
            l2_gbs = l2_by / (hbm["spmm"]["ms_per_step"] * 1e-3) / 1e9
            hbm["spmm"].update({"bound": "l2", "l2_gathered_bytes_per_step": l2_by, "l2_achieved_gbs": l2_gbs,
                                "l2_peak_gbs": l2_peak_gbs, "l2_frac": l2_gbs / l2_peak_gbs,
                                "l2_peak_source": "live cggm_test_l2_peak (16-byte loads over a 24 MB L2-resident "
                                                  "buffer, every SM)"})

    # ---------------------------------------------------------------- e2e through the public API
    e2e = None
    from paper_1509_04681_b200 import HostCsc, host_colmajor
    if not args.no_e2e and world == 1:
        # the public host-buffer entry point: X, Y and the CSCs from page-locked host memory, uploaded
        # by the library (Lambda first, the factorisation overlapping the X / Y transfers), S_yy formed
        # in the call, the scalar results read back (grad_Theta streamed when the bench streams it)
        Xh, Yh = host_colmajor(P.X), host_colmajor(P.Y)
        Lh, Thh = HostCsc.from_host(lam_h), HostCsc.from_host(th_h)
        h2d = (Xh.numel() + Yh.numel()) * 8 + sum(t.numel() * t.element_size() for c_ in (Lh, Thh)
                                                  for t in (c_.colptr, c_.rowidx, c_.val))
        d2h = ctypes.sizeof(_abi.cggm_objective_out) + ctypes.sizeof(_abi.cggm_active_out) + 8 + 4 + 8
        Syy_e = colmajor_empty(P.q, P.q)
        e2e_bufs = dict(bufs)

        def step_e2e():
            return ctx.cggm_newton_eval_host(Xh, Yh, Lh, Thh, P.lam_L, P.lam_T, True, bufs=e2e_bufs, Syy=Syy_e,
                                             stream_grad_theta=args.stream_grad_theta)

        step_e2e()
        step_e2e()
        e2_steps = max(1, min(args.steps, 3))
        e2ms = timed(step_e2e, e2_steps)
        e2e = {"value": e2_steps / (e2ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": e2_steps,
               "includes": "cggm_newton_eval_host: H2D of X, Y, Lambda, Theta from page-locked host memory "
                           "(overlapped with the factorisation) + S_yy + evaluation + D2H of scalars"
                           + ("; grad_Theta streamed (not stored)" if args.stream_grad_theta else "")}
    elif not args.no_e2e:
        # N > 1: every rank uploads its row block of X and Y and the two CSCs from page-locked host
        # memory each step, evaluates through the sharded evaluator (library calls + collectives) and
        # reads the objective back
        Xh, Yh = host_colmajor(P.X[a:b]), host_colmajor(P.Y[a:b])
        Lh, Thh = HostCsc.from_host(lam_h), HostCsc.from_host(th_h)
        h2d = (Xh.numel() + Yh.numel()) * 8 + sum(t.numel() * t.element_size() for c_ in (Lh, Thh)
                                                  for t in (c_.colptr, c_.rowidx, c_.val))

        def step_e2e():
            X.copy_(Xh, non_blocking=True)
            Y.copy_(Yh, non_blocking=True)
            for dc, hc in ((Lam, Lh), (Th, Thh)):
                for f_ in ("colptr", "rowidx", "val"):
                    getattr(dc, f_).copy_(getattr(hc, f_), non_blocking=True)
            r_ = ev.evaluate(X, Y, Lam, Th, P.lam_L, P.lam_T, True)
            return float(r_["f"])

        step_e2e()
        e2_steps = max(1, min(args.steps, 3))
        e2ms = timed(step_e2e, e2_steps)
        e2e = {"value": e2_steps / (e2ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 8, "steps": e2_steps,
               "includes": "per rank: H2D of its X / Y row block and the Lambda / Theta CSCs from page-locked "
                           "host memory + the sharded evaluation + D2H of f; max over ranks"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(P)
    barrier()
    fp32 = None
    if world == 1 and not args.no_fp32 and args.config == "large":
        del bufs
        ctx.lib.cggm_ctx_release_workspace(ctx.h)
        torch.cuda.empty_cache()
        fp32 = fp32_variant(["medium", "large"], max(3, min(args.steps, 5)), P_large=P)

    res = last
    obj = res["objective"] if world == 1 else {"f": res["f"]}
    step_achieved = all_flops / (ms_step * 1e-3) / world / 1e12
    if rank == 0:
        roof = {"bound": "tensor", "kernel": "gemm_dmma_kernel family (FP64 DMMA.8x8x4): every dense contraction "
                                             "of the step (97% of its time)",
                "achieved": step_achieved, "peak": peak_tflops, "unit": "TFLOP/s", "frac": step_achieved / peak_tflops,
                "traffic": _dominant_traffic(),
                "measured_in": f"timed region A: all algorithmic flops of the step ({all_flops:.4g}) / "
                               f"({world} GPU x {ms_step:.2f} ms)",
                "peak_source": f"live DMMA.8x8x4 microbenchmark on this GPU ({args.peak_seconds:.1f} s, "
                               "2 CTAs/SM); MEASURED_PEAKS.json has no FP64 entry",
                "traffic_source": "dram read+write bytes per launch of the largest launch (X^T E) from the "
                                  "committed ncu --set full capture"}
        if world == 1:
            gemm_ms = sum(phases[t]["ms_per_step"] for t in GEMM_TAGS if t in phases)
            roof["attribution_pass_b"] = {
                "gemm_ms_per_step": gemm_ms, "gemm_alg_flops_per_step": gemm_flops,
                "gemm_tflops": gemm_flops / (gemm_ms * 1e-3) / 1e12,
                "gemm_frac": gemm_flops / (gemm_ms * 1e-3) / 1e12 / peak_tflops,
                "lauum_tflops": phases.get("lauum", {}).get("tflops"),
                "what": f"serialised separate calls without lookahead, per-launch CUDA events, {prof_steps} steps "
                        f"({prof_elapsed / prof_steps:.1f} ms/step); per-launch durations include the "
                        f"latency-bound bottom of the recursions, so they sum to more than the overlapped step"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.config, "n": P.n, "p": P.p, "q": P.q, "nnz_theta": P.theta_star.nnz,
                       "nnz_lambda": P.lam_star.nnz, "lambda": P.lam_L, "point": "generating (Lambda*, Theta*)",
                       "parallelism": (f"sample-shard dp{world}, " + ("distributed inverse and trial factorisation" if dist_inv else
                                       "rank-0 inverse + split objective") + f", {args.allreduce} all-reduce, grad_Theta "
                                       f"{args.grad_theta}") if world > 1 else "1 GPU",
                       "l2": l2_note(P),
                       "setup_syy_ms": setup_ms, "generator_s": round(t_gen, 2),
                       "grad_theta": "streamed into the active sets (not stored)" if args.stream_grad_theta
                       else "stored (p x q)"},
            "clocks": clk_all[0] if world == 1 else {**(clk_all[0] or {}), "per_rank": clk_all},
            "step_ms_distribution": step_dist,
            "step_variants": variants,
            "env": run_env(),
            "gpu_launches": int(sum(launches_all)),
            "gpu_launches_per_rank": launches_all if world > 1 else None,
            "roofline": roof,
            "phases": phases if world == 1 else None,
            "comm": comm,
            "hbm_roofline": {"peak_gbs": HBM_PEAK_GBS, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)",
                             "kernels": hbm} if world == 1 else None,
            "e2e": e2e,
            "factor_reuse": reuse,
            "fp32": fp32,
            "cpu_baseline": cpu,
            "result": {"f": obj.get("f"), "logdet": res.get("logdet"),
                       "m_L": res["active"]["m_L"], "m_T": res["active"]["m_T"],
                       "subgrad_l1": res["active"]["subgrad_l1"]},
        }
        if functional:
            line["functional_only"] = "all ranks on one GPU (CGGM_BENCH_DEVICE): not a measurement"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
