#!/usr/bin/env python
"""bench.py -- OCSC training images/sec on B200 (BASELINE.json metric), one JSON line.

Headline workload (BASELINE.json configs[1]): seeded synthetic 32x32 images
zero-padded to 42x42, K = 100 filters of 11x11, beta = 1, rho_code = rho_dict = 1, J = 10
dictionary rounds, <= 300 code iterations, float32 arithmetic (float64 history), global
mini-batch 50.  A step is one mini-batch through the whole hot path: batched code ADMM ->
objective -> history fold -> inverse / Cholesky -> J dictionary rounds.  At N = 1 the line also
carries a "secondary" block with BASELINE configs 2 and 3 (training steps, same contract) and
config 4 at K = 256 (history accumulation + Cholesky solve), measured in the same run.

    python bench.py [--gpus N --steps K --warmup W]            # this build
    python bench.py --impl reference [--steps K --warmup W]    # CPU reference arm (oracle port)
    torchrun --nproc-per-node N bench.py --gpus N ...          # N > 1: strong scaling

Scaling is strong: the global mini-batch of the configuration is split into ragged sample shards
(50 over 8 ranks = 7,7,6,6,6,6,6,6), so the dictionary is updated once per B samples at every N.

Timing: W untimed warm-up steps, then K steps each bracketed by CUDA events on the trainer's
stream, L2 flushed (256 MiB write) between steps outside the events, barrier + synchronize
around the block, max over ranks.  `value` has the inputs already resident in HBM; `e2e` runs
the public API (`OnlineTrainer.partial_fit`) on pinned host arrays, H2D of the images and D2H
of the per-sample objectives inside the timed region.  The roofline's kernel time comes from
CUDA events the trainer records around its code kernels inside the timed steps.
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

METRIC = "OCSC training images/sec at 1/2/4/8 B200; % of HBM/FP32 roofline per kernel"
UNIT = "images/s"
# BASELINE.json training configs; config 1 is the headline, 2 and 3 ride along as
# the line's "secondary" block (or run alone with --config N)
TRAIN_CFGS = {
    1: (dict(dims0=(32, 32), grid=(42, 42), fdims=(11, 11), K0=20, K=100, beta=1.0, rho_code=1.0, rho_dict=1.0,
             J=10, max_iters=300, rel_tol=1e-3, B=50),
        "BASELINE config 1: seeded synthetic 32x32 images zero-padded to 42x42, K=100 filters 11x11, beta=1, "
        "rho=1, J=10, <=300 code iterations, float32 (history float64), global mini-batch 50"),
    2: (dict(dims0=(100, 100), grid=(100, 100), fdims=(11, 11), K0=20, K=100, beta=1.0, rho_code=1.0,
             rho_dict=1.0, J=10, max_iters=300, rel_tol=1e-3, B=10),
        "BASELINE config 2: seeded synthetic 100x100 images (no padding), K=100 filters 11x11, beta=1, rho=1, "
        "J=10, <=300 code iterations, float32 (history float64), global mini-batch 10"),
    3: (dict(dims0=(256, 256), grid=(266, 266), fdims=(11, 11), K0=64, K=256, beta=0.5, rho_code=1.0,
             rho_dict=1.0, J=10, max_iters=300, rel_tol=1e-3, B=32, history="float32"),
        "BASELINE config 3: seeded synthetic 256x256 images zero-padded to 266x266, K=256 filters 11x11, "
        "beta=0.5, rho=1, J=10, <=300 code iterations, float32 with the complex64 history BASELINE sizes "
        "(9.4 GB packed half spectrum), global mini-batch 32"),
}


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def make_images(cfg, n, start, seed=0):
    from paper_1706_06972_b200.workloads import synth_images  # seeded inputs
    return synth_images(n, cfg["dims0"], cfg["grid"], cfg["K0"], filter_dims=cfg["fdims"], seed=seed,
                        start=start).reshape(n, -1)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks/throttle reasons every 20 ms; `stop()` summarises the samples that
    arrived inside the marked window(s) (the timed region), so idle samples before/after it
    do not dilute the median."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index, interval_ms=20):
        self.gpu = gpu_index
        self.interval = interval_ms
        self.rows = []      # (host time, fields)
        self.windows = []   # (t0, t1) host times of timed regions
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.interval)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append((time.perf_counter(), parts))

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        inside = [r for t, r in self.rows if any(a <= t <= b for a, b in self.windows)]
        rows = inside or [r for _, r in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = [x for x in (num(r[0]) for r in rows) if x is not None]
        mx = [x for x in (num(r[1]) for r in rows) if x is not None]
        pw = [x for x in (num(r[6]) for r in rows) if x is not None]
        reasons = sorted({n for r in rows for n, v in zip(self.NAMES, r[2:6]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "in_timed_region": bool(inside),
                "power_w_median": statistics.median(pw) if pw else None}


def fp32_peak_tflops(sms, sm_mhz):
    """(peak, source): the measured FMA-chain rate (profiles/r1_fma_peaks.json, scripts/fma_peak.cu)
    scaled to the clock the kernel ran at; the nominal 128 FMA/clk/SM if the file is absent."""
    try:
        m = json.load(open(os.path.join(ROOT, "profiles", "r1_fma_peaks.json")))
        per_clk = float(m["ffma_tflops"]) * 1e12 / (int(m["sms"]) * float(m["sm_mhz"]) * 1e6)
        return (sms * per_clk * float(sm_mhz) * 1e6 / 1e12,
                f"measured FFMA chain rate ({per_clk:.0f} flop/clk/SM, profiles/r1_fma_peaks.json, "
                f"scripts/fma_peak.cu) x median SM clock in the timed region")
    except (OSError, KeyError, ValueError):
        return sms * 128 * 2 * float(sm_mhz) * 1e6 / 1e12, "nominal 128 FMA/clk/SM x 2 x median SM clock"


# --------------------------------------------------------------- CPU legs --
def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_description():
    """Host CPU model, thread settings and numpy / BLAS versions."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = []
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": i.get("internal_api"), "version": i.get("version"), "threads": i.get("num_threads")}
                for i in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "numpy": np.__version__, "blas": blas,
            "env": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")},
            "note": "numpy FFTs (pocketfft) are single-threaded; the batched inverse/einsum parts use the BLAS threads"}


def cpu_oracle_rate(cfg, n_images, budget_s=None, warmup=0):
    """Images/s of the CPU reference algorithm (oracle port, OnlineTrainer.step = mini-batch of 1)."""
    from oracle import ocsc_oracle as O
    tr = O.Trainer(cfg["grid"], cfg["fdims"], K=cfg["K"], beta=cfg["beta"], rho_code=cfg["rho_code"],
                   rho_dict=cfg["rho_dict"], inner_iters=cfg["J"], seed=0, code_max_iters=cfg["max_iters"],
                   code_rel_tol=cfg["rel_tol"], stop_tol=0.0)
    X = make_images(cfg, n_images + warmup, start=10_000_000)
    for i in range(warmup):
        tr.step_batch(X[i:i + 1])
    done, t0 = 0, time.perf_counter()
    for i in range(warmup, warmup + n_images):
        tr.step_batch(X[i:i + 1])
        done += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt, done, dt


def run_reference(args, rank):
    if rank != 0:
        return
    cfg, workload = TRAIN_CFGS[args.config]
    budget = float(os.environ.get("OCSC_REF_BUDGET_S", "150"))
    rate, done, dt = cpu_oracle_rate(cfg, args.steps, budget_s=budget, warmup=min(args.warmup, 1))
    cores = cpu_threads()
    sample = (f"{done} timed step(s) of 1 image each of config {args.config} (reference OnlineTrainer.step "
              f"semantics, oracle/ocsc_oracle.py numpy port, float64), {dt:.1f} s; warm-up {min(args.warmup, 1)} step")
    line = {"metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": done, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * dt / max(done, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded planted-dictionary images, SURVEY.md 8(d))",
            "config": {"workload": workload, "global_batch": 1, "parallelism": "cpu (BLAS threads)"},
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                             "host": cpu_description()},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU legs --
def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "MEASURED_PEAKS.json (driver-measured)"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback 6650 GB/s (B200_PROFILING.md)"


def load_traffic():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        return {}


def code_intervals(tl):
    """(start, end) events of the code-ADMM kernels per step from the trainer's timeline marks
    (fused: main + tail launches; stream / cuFFT: the whole coding loop)."""
    out, start = [], None
    for label, ev in tl:
        if label in ("main start", "code start"):
            start = ev
        elif label in ("tail end", "code end") and start is not None:
            out.append((start, ev))
            start = None
    return out


def train_line(args, cfg_id, rank, world, local_rank, steps, warmup, e2e=True, cpu=True):
    """One training configuration through the public API; returns the JSON dict (rank 0)."""
    import torch
    import torch.distributed as dist

    import paper_1706_06972_b200 as ob
    from paper_1706_06972_b200 import _lib
    from paper_1706_06972_b200.sharded import DistComm, ShardedTrainer, sample_shards

    cfg, workload = TRAIN_CFGS[cfg_id]
    dev = torch.device("cuda", local_rank)
    lib = _lib.load()
    B = args.batch if (args.batch and cfg_id == args.config) else cfg["B"]
    mine = sample_shards(B, world)[rank]
    b = mine.stop - mine.start
    shape = ob.SignalShape(cfg["grid"], cfg["fdims"])
    tcfg = ob.TrainConfig(n_filters=cfg["K"], beta=cfg["beta"], rho_code=cfg["rho_code"], rho_dict=cfg["rho_dict"],
                          inner_iters=cfg["J"], seed=0, code_max_iters=cfg["max_iters"], code_rel_tol=cfg["rel_tol"],
                          dtype="float32", history_dtype=cfg.get("history", "float64"), batch_size=B, stop_tol=0.0,
                          poll=16)
    Trainer = (lambda: ShardedTrainer(shape, tcfg, DistComm())) if world > 1 else (lambda: ob.OnlineTrainer(shape, tcfg))
    nsteps = warmup + steps
    P = shape.size
    # strong scaling: every step is one global mini-batch of B images; rank r codes its shard
    X = np.stack([make_images(cfg, B, start=s * B)[mine] for s in range(nsteps)]).astype(np.float32)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.2)

    # ---- value: inputs resident in HBM, device-timed --------------------------------
    trainer = Trainer()
    Xd = torch.as_tensor(X).to(dev)
    for s in range(warmup):
        trainer.partial_fit(Xd[s])
    torch.cuda.synchronize()
    barrier()
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    iters_sum, iters_max = [], []
    launches0 = lib.ocsc_kernel_launches()
    trainer._tl = []  # code-kernel start/end events inside the timed steps (the roofline's timer)
    torch.cuda.synchronize()
    barrier()
    t_on = time.perf_counter()
    for i in range(steps):
        flush.zero_()
        evs[i][0].record(stream)
        res = trainer.partial_fit(Xd[warmup + i])
        evs[i][1].record(stream)
        iters_sum.append(int(np.sum(res.iterations)))
        iters_max.append(int(np.max(res.iterations)) if len(res.iterations) else 0)
    torch.cuda.synchronize()
    sampler.mark(t_on, time.perf_counter())
    barrier()
    launches = lib.ocsc_kernel_launches() - launches0
    path = trainer.last_path
    total_ms = max_over_ranks(sum(a.elapsed_time(b_) for a, b_ in evs))
    value = B * steps / (total_ms / 1e3)
    code_ms = [a.elapsed_time(b_) for a, b_ in code_intervals(trainer._tl)]
    trainer._tl = None
    code_ms_step = float(np.mean(code_ms)) if code_ms else float("nan")

    # ---- e2e: public API, pinned host input, objectives back to host -----------------
    e2e_line = None
    if e2e:
        del trainer
        torch.cuda.empty_cache()
        trainer2 = Trainer()
        Xh = torch.as_tensor(X).pin_memory()
        for s in range(warmup):
            trainer2.partial_fit(Xh[s])
        torch.cuda.synchronize()
        barrier()
        e2e_s = 0.0
        for i in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r2 = trainer2.partial_fit(Xh[warmup + i])
            _ = float(r2.objectives.sum())
            t1 = time.perf_counter()
            sampler.mark(t0, t1)
            e2e_s += t1 - t0
        barrier()
        e2e_s = max_over_ranks(e2e_s)
        e2e_line = {"value": B * steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": b * P * 4,
                    "d2h_bytes_per_step": (2 * b + 4) * 8}
        del trainer2
    else:
        del trainer
    torch.cuda.empty_cache()
    clocks = sampler.stop()

    # ---- roofline of the dominant kernel: the code ADMM of the step ------------------------
    peaks, peak_src = load_peaks()
    sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    fp32_peak, fp32_src = fp32_peak_tflops(torch.cuda.get_device_properties(dev).multi_processor_count, sm_mhz)
    H, W = cfg["grid"]
    Pf, Ph, K, s = H * W, H * (W // 2 + 1), cfg["K"], 4
    flops_img_iter = 2 * K * 2.5 * Pf * np.log2(Pf) + 16 * Ph * K + 8 * Pf * K
    bytes_img_iter = 8 * Pf * K * s + 8 * Ph * K * s
    flops_step = float(np.mean(iters_sum)) * flops_img_iter
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tj = load_traffic()
    on_chip = path in ("fused", "fused+split") or (path and path.startswith("stream") and (H, W) == (100, 100))
    kname = {"fused": "k_code_fused (one cluster per sample, ADMM state in SMEM)",
             "fused+split": "k_code_fused main + tail launches (one cluster per sample, ADMM state in SMEM)"}.get(
        path, "k_plane (one CTA per (sample, filter group), planes in SMEM) + k_gsum per iteration"
        if on_chip else "k_rows + k_cols_f + k_gsum + k_cols_i per iteration (state streamed through HBM)")
    it_ms = code_ms_step / max(float(np.mean(iters_max)), 1.0)
    traffic_key = ("fused_bytes_per_batch_iter" if path and path.startswith("fused") else
                   f"plane{H}_bytes_per_batch_iter" if on_chip else f"stream{H}_bytes_per_batch_iter")
    traffic = tj.get(traffic_key)
    if on_chip:
        achieved = flops_step / (code_ms_step / 1e3) / 1e12
        roof = {"bound": "fp32", "kernel": kname, "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": achieved / fp32_peak, "traffic": traffic,
                "algorithmic": "SURVEY 8(d) flops 2K*2.5*P*log2(P) + 16*Ph*K + 8*P*K per image-iteration x the "
                               "iterations each sample ran",
                "peak_source": fp32_src, "code_ms_per_step": code_ms_step, "iter_ms": it_ms,
                "timer": "CUDA events on the launching streams around the code kernels of every timed step",
                "hbm_equivalent": {"achieved_GB/s": float(np.mean(iters_sum)) * bytes_img_iter / code_ms_step / 1e6,
                                   "peak": hbm, "note": "SURVEY 8(d) G1-G4 bytes an HBM-streaming design would "
                                   "move; this kernel keeps the state on chip (traffic = measured DRAM bytes per "
                                   "mini-batch iteration)"}}
        pipe = tj.get("fused_ncu_set_full") if path.startswith("fused") else None
        if pipe:
            roof["ncu_fma_pipe_active_pct"] = pipe.get("sm__pipe_fma_cycles_active_pct_of_peak_active")
            roof["ncu_source"] = pipe.get("source")
    else:
        achieved = (traffic or float("nan")) / (it_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic,
                "algorithmic": "measured DRAM bytes (ncu) of one mini-batch iteration of the streaming kernels "
                               "(profiles/traffic.json)", "peak_source": peak_src, "code_ms_per_step": code_ms_step,
                "iter_ms": it_ms, "fp32_equivalent": {"achieved_TFLOP/s": flops_step / code_ms_step / 1e9,
                                                       "peak": fp32_peak}}

    # ---- CPU baseline (rank 0, N = 1 only) -------------------------------------------
    cpu_line = None
    if cpu and rank == 0 and world == 1 and not args.no_cpu_baseline:
        if cfg_id == 3:
            cpu_line = {"value": None, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                        "sample": "n/a (memory): the reference's inv_gram for config 3 alone is 74 GB of complex128 "
                                  "(dictionary.py:30-54), plus >= 3 same-size temporaries in update_history"}
        else:
            n = int(os.environ.get("OCSC_CPU_SAMPLE_IMAGES", "3" if cfg_id == 1 else "1"))  # ~12 s of CPU work
            rate, done, dt = cpu_oracle_rate(cfg, n)
            cpu_line = {"value": rate, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                        "sample": f"{done} image(s) of config {cfg_id} through oracle/ocsc_oracle.py (reference "
                                  f"algorithm, OnlineTrainer.step semantics, float64), {dt:.1f} s on host cores",
                        "host": cpu_description()}

    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": total_ms / steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded planted-dictionary images, SURVEY.md 8(d))",
            "config": {"workload": workload, "global_batch": B, "per_rank_batch": b, "path": path,
                       "code_iterations_mean": float(np.mean(iters_sum)) / max(b, 1),
                       "l2": "flushed between timed steps (256 MiB device write outside the events)",
                       "parallelism": (f"dp{world} x freq{world}: the global mini-batch of {B} split into ragged "
                                       f"sample shards, history and dictionary ADMM sharded by spectrum rows "
                                       f"(all_to_all of code spectra + K x M all-reduce per round)" if world > 1 else
                                       "single GPU")},
            "roofline": roof, "cpu_baseline": cpu_line, "e2e": e2e_line, "gpu_launches": int(launches),
            "clocks": clocks}


def run_b200(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank)
    line = train_line(args, args.config, rank, world, local_rank, args.steps, args.warmup)
    if args.config == 1 and (world == 1 or args.secondary) and not args.no_secondary:
        # the other BASELINE configurations in the same run (driver-visible)
        sec = {}
        for cid, st, wu in ((2, 5, 2), (3, 2, 1)):
            try:
                sec[f"config{cid}"] = train_line(args, cid, rank, world, local_rank, st, wu, e2e=(cid == 2),
                                                 cpu=False)
            except Exception as e:  # a secondary failure must not lose the headline
                sec[f"config{cid}"] = {"error": f"{type(e).__name__}: {e}"}
        try:
            args_k = argparse.Namespace(**vars(args))
            args_k.ks, args_k.steps, args_k.warmup = [256], 3, 1
            sec["config4_K256"] = run_history_microbench(args_k, rank, world, local_rank, emit=False)[0]
        except Exception as e:
            sec["config4_K256"] = {"error": f"{type(e).__name__}: {e}"}
        line["secondary"] = sec
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_history_microbench(args, rank, world, local_rank, emit=True):
    """BASELINE config 4: per-frequency rank-64 history accumulation + (A + rho I) Cholesky solve.

    P = 128 x 128 independent frequencies (full grid: random codes are not Hermitian),
    complex64, z ~ CN(0,1) and x ~ CN(0,1) seeded, rho = 1 (plain ridge on the summed A),
    one right-hand side per frequency (the accumulated cross term).  Bytes/flops per
    SURVEY.md 8(d): G6 and G7 formulas.
    """
    import torch

    import paper_1706_06972_b200 as ob
    from paper_1706_06972_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    _lib.load()
    P, B, s = 128 * 128, 64, 4
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    fp32, _ = fp32_peak_tflops(torch.cuda.get_device_properties(dev).multi_processor_count, 1965.0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    shape = ob.SignalShape((P,), (1,))
    lines = []
    for K in args.ks:
        z = torch.complex(torch.randn(B, P, K, device=dev, generator=gen),
                          torch.randn(B, P, K, device=dev, generator=gen)) / np.sqrt(2)
        x = torch.complex(torch.randn(B, P, device=dev, generator=gen),
                          torch.randn(B, P, device=dev, generator=gen)) / np.sqrt(2)
        zero = torch.zeros(P, K, dtype=torch.complex64, device=dev)
        out = torch.empty_like(zero)
        times = {"accumulate": [], "factor": [], "solve": []}
        for rep in range(args.warmup + args.steps):
            h = ob.HistoryState(shape, K, 1.0 / P, dtype=torch.complex64, solver="chol")  # ridge rho*P = 1
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            torch.cuda.synchronize()
            ev[0].record()
            h.accumulate(z, (P * K, 1, K), x, (P, 1), B)
            ev[1].record()
            h.count = 1  # plain ridge rho = 1 on the summed A (t * rho * P with t = 1)
            h.factor(check=False)
            ev[2].record()
            h.rowsolve(zero, zero, 1, K, out, check=False)
            ev[3].record()
            torch.cuda.synchronize()
            if rep >= args.warmup:
                times["accumulate"].append(ev[0].elapsed_time(ev[1]))
                times["factor"].append(ev[1].elapsed_time(ev[2]))
                times["solve"].append(ev[2].elapsed_time(ev[3]))
            del h
        # parity on a few frequencies against a dense complex128 solve
        zz = z[:, :4].cpu().numpy().astype(np.complex128)
        xx = x[:, :4].cpu().numpy().astype(np.complex128)
        ref = []
        for p in range(4):
            A = np.einsum("bi,bj->ij", zz[:, p], zz[:, p].conj()) + np.eye(K)
            ref.append(np.conj(np.linalg.solve(A, np.einsum("b,bk->k", xx[:, p].conj(), zz[:, p]))))
        ref = np.array(ref)
        err = float(np.linalg.norm(out[:4].cpu().numpy() - ref) / np.linalg.norm(ref))
        npk = K * (K + 1) / 2
        g6_bytes = 2 * P * npk * 2 * s + B * P * (K + 1) * 2 * s
        g6_flops = 4 * K * (K + 1) * B * P
        g7_bytes = 2 * P * npk * 2 * s + 2 * P * K * 2 * s
        g7_flops = (4 / 3) * K ** 3 * P + 8 * K * K * P
        ta, tf, ts = (min(times[k]) for k in ("accumulate", "factor", "solve"))
        line = {"metric": "history accumulation + Cholesky solve (BASELINE config 4)", "K": K, "P": P, "B": B,
                "dtype": "c64", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms": {"accumulate": ta, "factor": tf, "solve": ts, "total": ta + tf + ts},
                "accumulate": {"GB/s": g6_bytes / ta / 1e6, "GFLOP/s": g6_flops / ta / 1e6,
                               "frac_hbm": g6_bytes / ta / 1e6 / hbm, "frac_fp32": g6_flops / ta / 1e9 / fp32},
                "cholesky_solve": {"GB/s": g7_bytes / (tf + ts) / 1e6, "GFLOP/s": g7_flops / (tf + ts) / 1e6,
                                   "frac_hbm": g7_bytes / (tf + ts) / 1e6 / hbm,
                                   "frac_fp32": g7_flops / (tf + ts) / 1e9 / fp32},
                "peaks": {"hbm_GB/s": hbm, "fp32_TFLOP/s_nominal": fp32},
                "parity_rel_err_vs_dense_c128": err, "data": "synthetic CN(0,1), seeded"}
        lines.append(line)
        if rank == 0 and emit:
            print(json.dumps(line), flush=True)
        del z, x
    return lines


def run_preprocess_microbench(args, rank, world, local_rank):
    """grayscale + LCN + edge taper (preprocessing.py:92-100), one fused launch.

    N = 1024 seeded RGB uint8 256 x 256 images (Flower/CIFAR-style stream, synthetic), float32 out
    (what the float32 trainer consumes).  Input 201 MB + output 268 MB > L2, so no flush is needed.
    Algorithmic bytes per image = H*W*3 (u8 in) + H*W*4 (f32 out).
    """
    import torch

    import paper_1706_06972_b200 as ob
    from paper_1706_06972_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    _lib.load()
    N, H, W = 1024, 256, 256
    rng = np.random.default_rng(2024 + rank)
    host = torch.from_numpy(rng.integers(0, 256, size=(N, H, W, 3), dtype=np.uint8)).pin_memory()
    imgs = host.to(dev)
    spec = ob.PreprocessSpec(seed=rank * N)
    out = ob.preprocess_batch(imgs, spec, out_dtype=torch.float32)
    torch.cuda.synchronize()
    hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    l0 = _lib.load().ocsc_kernel_launches()
    times = []
    for rep in range(args.warmup + args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = ob.preprocess_batch(imgs, spec, out_dtype=torch.float32)
        b.record()
        torch.cuda.synchronize()
        if rep >= args.warmup:
            times.append(a.elapsed_time(b))
    launches = (_lib.load().ocsc_kernel_launches() - l0) * args.steps // (args.warmup + args.steps)
    e2e_t = []
    res = torch.empty((N, H, W), dtype=torch.float32).pin_memory()
    for rep in range(args.warmup + args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        o = ob.preprocess_batch(host.to(dev, non_blocking=True), spec, out_dtype=torch.float32)
        res.copy_(o, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        if rep >= args.warmup:
            e2e_t.append(a.elapsed_time(b))
    from oracle import ocsc_oracle as O

    ref = O.preprocess(host[0].numpy().astype(np.float64), seed=spec.seed)
    err = float(np.abs(res[0].double().numpy() - ref).max() / np.abs(ref).max())
    t0 = time.perf_counter()
    for i in range(4):
        O.preprocess(host[i].numpy().astype(np.float64), seed=spec.seed + i)
    cpu_ips = 4 / (time.perf_counter() - t0)
    ms = float(np.median(times))
    algo = N * H * W * (3 + 4)
    flops = N * H * W * (8 * spec.lcn_window + 4 * spec.taper_size + 10)
    fp64 = 148 * 64 * 2 * 1965e6 / 1e12
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get("preprocess_dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    line = {"metric": "preprocessed images/s (grayscale + LCN + edge taper, SURVEY 8(f) f4)",
            "value": N * world / (ms / 1e3), "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "dtype": "f64 arithmetic, u8 in, f32 out", "data": "synthetic RGB uint8, seeded",
            "config": {"workload": f"{N} RGB {H}x{W} images per GPU per step", "l2": "working set > L2"},
            "roofline": {"bound": "fp64", "kernel": "k_preprocess<uint8_t, float, 9, 11>",
                         "achieved": flops / ms / 1e9, "peak": fp64, "unit": "TFLOP/s", "frac": flops / ms / 1e9 / fp64,
                         "traffic": traffic, "algorithmic_flops_per_launch": flops,
                         "flops_note": "per pixel 8*window (LCN: 2 passes x {x, x^2}) + 4*taper (2 passes) + 10 "
                                       "(normalise, blend); float64 is the reference's arithmetic",
                         "peak_source": "148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz (nominal; not in MEASURED_PEAKS)",
                         "hbm": {"algorithmic_bytes": algo, "achieved_GB/s": algo / ms / 1e6, "peak": hbm,
                                 "frac": algo / ms / 1e6 / hbm}},
            "cpu_baseline": {"value": cpu_ips, "unit": "images/s", "cores": 1, "kind": "port",
                             "sample": "4 images through oracle/ocsc_oracle.py preprocess (numpy, float64)"},
            "e2e": {"value": N / (float(np.median(e2e_t)) / 1e3), "unit": "images/s",
                    "h2d_bytes_per_step": N * H * W * 3, "d2h_bytes_per_step": N * H * W * 4},
            "gpu_launches": int(launches), "parity_max_rel_err_vs_oracle_f32_out": err}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", type=int, default=1, choices=[1, 2, 3, 4, 5],
                    help="1: BASELINE config 1 training step (default); 2, 3: BASELINE configs 2 and 3; "
                         "4: history + Cholesky microbenchmark; 5: image preprocessing (row f4)")
    ap.add_argument("--ks", type=int, nargs="+", default=[64, 128, 256, 512], help="K values for --config 4")
    ap.add_argument("--no-secondary", action="store_true", help="headline config 1 only (no configs 2-4 block)")
    ap.add_argument("--secondary", action="store_true", help="also run the secondary block at N > 1")
    args = ap.parse_args()
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if os.environ.get("OCSC_BENCH_BACKEND", "nccl") != "nccl":
        import torch
        local_rank %= max(torch.cuda.device_count(), 1)
    if args.impl == "reference":
        if args.config not in TRAIN_CFGS:
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "the reference arm times training configs 1-3"}))
            return
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        # OCSC_BENCH_BACKEND=gloo is a functional check of the N > 1 code path on a box with fewer
        # GPUs than ranks (host-staged collectives; never a reported number)
        backend = os.environ.get("OCSC_BENCH_BACKEND", "nccl")
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # NVLS / transport selection in the log (stderr)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        if args.config == 4:
            run_history_microbench(args, rank, world, local_rank)
            return
        if args.config == 5:
            run_preprocess_microbench(args, rank, world, local_rank)
            return
        run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
