#!/usr/bin/env python
"""bench.py -- fwd and fwd+bwd signature throughput (paths/s) on 1..8 B200s.

One JSON line on rank 0 (the driver's contract).  A "step" is one pass of the
hot path over one batch: the forward Chen kernel (S_{0,T} of every word) and
the memory-lean backward (dL/dX from S_{0,T} and a dense upstream), both
through the C ABI (include/sigkit_b200.h) on inputs already resident in HBM.

Workload (default): BASELINE.json config 5 -- truncated signature d=16,
depth 4 (W = 69,904 words), L = 512 samples, fp32, ONE batch of 65,536 paths
split across the ranks (strong scaling: rank r owns
``sharding.shard_range(65536, r, N)``; the batch axis shards with no
collective).  ``--weak`` gives every rank the config's whole batch instead;
``--config c1|c2|c3|c4`` measures another BASELINE config on the same harness.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (one process per GPU, NCCL), so
``python bench.py --gpus 8`` and the driver's torchrun launch are the same run.

Extra keys:
  fwd          forward-only paths/s (the metric's first half)
  roofline     the dominant kernel (backward Chen kernel) against the FP32
               FMA pipe: algorithmic flop per launch / CUDA-event duration
               (frac = frac_alg); frac_min_work credits only
               the shared-Horner T-node FMAs the kernels must execute;
               ncu_exec carries the executed FMA-pipe (and tensor-pipe) share
               from the committed profiles/ capture
  roofline_fwd the same for the forward Chen kernel
  e2e          fwd+bwd paths/s through the public autograd API with the
               paths copied from pinned host memory and dL/dX + the loss
               read back every step
  e2e_fwd      forward paths/s through the numpy drop-in signature_forward
               (host array in, host array out)
  cpu_baseline the CPU oracle port (oracle/, a restatement of the reference
               numba kernels) on this host's cores, bounded sample, N=1 only
  clocks       nvidia-smi SM clocks / throttle reasons sampled during the
               timed region

``--impl reference`` times the reference algorithm on the host cores instead
(the oracle port; the reference is a numba package that cannot travel to the
GPU box) and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fwd and fwd+bwd signature throughput (paths/sec) at 1/2/4/8 B200"
FP32_LANES_PER_SM = 128
FP64_LANES_PER_SM = 64


def parse_args(argv=None):
    p = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--config", default="c5", choices=("c1", "c2", "c3", "c4", "c5", "p1", "p2"),
                   help="BASELINE.json configs c1-c5; p1/p2 = pathsig's H200 training rows (PAPER.md:429-449)")
    p.add_argument("--precision", default="config", choices=("config", "fp64"),
                   help="fp64: run the config in float64 (the reference's backward contract, backward.py:166-167)")
    p.add_argument("--batch", type=int, default=0, help="override the per-rank batch (profiling only)")
    p.add_argument("--weak", action="store_true", help="every rank runs the config's whole batch (weak scaling)")
    p.add_argument("--strong", action="store_true", help="(default) shard one fixed global batch across the ranks")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-split", type=int, default=8,
                   help="max sub-batches per e2e step (copy/compute pipeline; each >= 256 paths)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--gather", action="store_true", help="also time the optional NCCL all-gather of S")
    p.add_argument("--policy", type=int, default=0, help="0 auto kernels, 1 generic trie kernels only")
    return p.parse_args(argv)


# -- helpers ---------------------------------------------------------------------------


def load_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


def fma_peak_tflops(dtype: str, sms: int, peaks: dict) -> tuple[float, str]:
    """FMA-pipe peak for the roofline: SMs x lanes x 2 flop x clock.

    MEASURED_PEAKS.json (driver-written) holds HBM copy bandwidth, bf16 GEMM and
    the SM max clock, not an FMA-pipe figure, so the peak is the pipe width
    times its ``sm_max_mhz`` (148 x 128 x 2 x 1965 MHz = 74.45 TF fp32,
    37.22 TF fp64), the SM count read from the device.
    """
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    lanes = FP32_LANES_PER_SM if dtype == "fp32" else FP64_LANES_PER_SM
    src = "MEASURED_PEAKS.json sm_max_mhz" if "sm_max_mhz" in peaks else "B200_PROFILING.md clocks.max.sm"
    return sms * lanes * 2 * mhz * 1e6 / 1e12, (
        f"{sms} SMs x {lanes} {dtype} FMA lanes x 2 flop x {mhz:.0f} MHz ({src})")


def ubench_peak_tflops(dtype: str) -> float | None:
    """The FFMA/DFMA pipe as tools/ubench_fma --peak measures it on this GPU (context only)."""
    exe = os.path.join(ROOT, "tools", "ubench_fma")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe, "--peak"], capture_output=True, text=True, timeout=60).stdout
        v = json.loads(out.strip().splitlines()[-1])["ffma_tflops" if dtype == "fp32" else "dfma_tflops"]
        return v if v > 0 else None
    except (OSError, ValueError, KeyError, IndexError, subprocess.TimeoutExpired):
        return None


def tf32_peak_tflops(peaks: dict) -> tuple[float, str]:
    """Dense tf32 tensor peak: half the measured dense bf16 rate (the tf32:bf16 ratio of
    B200_PROFILING.md's 1.1 / 2.25 PF), else the guide's 1.1 PF."""
    if peaks.get("bf16_tflops"):
        return peaks["bf16_tflops"] / 2.0, "MEASURED_PEAKS.json bf16_tflops / 2 (tf32 runs at half the bf16 rate)"
    return 1100.0, "B200_PROFILING.md dense tf32"


def ncu_exec(kernel: str, config: str) -> dict | None:
    """Executed-work view of `kernel` from the committed ncu capture (profiles/ncu_summary.json)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        ent = json.load(f).get(config, {}).get(kernel)
    if not ent:
        return None
    keys = ("fma_pipe_pct", "fp64_pipe_pct", "tensor_pipe_pct", "issue_active_pct", "warps_active_pct", "source")
    return {k: ent[k] for k in keys if ent.get(k) is not None}


def ncu_traffic(kernel: str, config: str) -> tuple[float | None, str | None]:
    """DRAM bytes per path of `kernel` from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        js = json.load(f)
    ent = js.get(config, {}).get(kernel)
    if not ent or not ent.get("paths"):
        return None, None
    return (ent["dram_read_bytes"] + ent["dram_write_bytes"]) / ent["paths"], ent.get("source")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md).

    The sampler starts before the timed region and waits for its first row, so
    nvidia-smi's start-up does not eat a short run; ``mark()`` brackets the timed
    region and only rows stamped inside it are summarised.
    """

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, enabled: bool, period_ms: int = 50):
        self.proc = None
        self.t0 = self.t1 = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        if enabled:
            try:
                os.makedirs(os.path.dirname(self.path), exist_ok=True)
                self.fh = open(self.path, "w")
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms",
                     str(period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
                import threading

                self.rows = []
                self.first = threading.Event()
                self.reader = threading.Thread(target=self._read, daemon=True)
                self.reader.start()
                self.first.wait(timeout=5.0)
            except (OSError, FileNotFoundError):
                self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.fh.write(line)
            self.rows.append((time.perf_counter(), line))
            self.first.set()

    def mark(self, start: bool) -> None:
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.reader.join(timeout=2)
        self.fh.close()
        rows = []
        t0 = self.t0 if self.t0 is not None else -math.inf
        t1 = self.t1 if self.t1 is not None else math.inf
        for ts, line in self.rows:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9 or not t0 <= ts <= t1:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[4]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": "timed region shorter than one nvidia-smi sample; raise --steps"}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows),
                "util_pct_median": statistics.median(r[2] for r in rows)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def workload(name: str, precision: str = "config"):
    from tests.configs import ALL_CONFIGS

    cfg = dict(ALL_CONFIGS[name])
    if precision == "fp64":
        cfg["dtype"] = np.float64
    return cfg


def sum_lengths(ws) -> int:
    return int(np.asarray(ws.lengths).sum())


def describe(name: str, cfg: dict, ws) -> str:
    kind = cfg["kind"]
    if kind == "truncated":
        s = f"truncated d={cfg['d']} depth={cfg['depth']}"
    elif kind == "custom":
        s = f"prefix-closed custom trie d={cfg['d']} (seeded, tests/golden/c3_words.json)"
    else:
        s = f"anisotropic d={cfg['d']} gamma={list(cfg['gamma'])} r={cfg['r']}"
    dt = "fp64" if cfg["dtype"] == np.float64 else "fp32"
    return f"{name}: {s}, W={len(ws)}, L={cfg['L']}, {dt}, fwd+bwd"


# -- CPU arm (oracle port of the reference numba kernels) ---------------------------------


def cpu_sample(name: str, cfg: dict, ws, threads: int, seed: int = 7):
    """Time the oracle port on a bounded sample of workload `name`.

    Forward on B_f = min(B, 2*threads) paths in the config dtype (the
    reference's mixed-precision fp32 path); backward on B_b = min(B, threads)
    paths in fp64 (the reference backward always upcasts, backward.py:166-167).
    Returns (fwd+bwd paths/s, fwd paths/s, t_f, t_b, B_f, B_b).
    """
    from oracle import oracle as ora  # the checker / CPU baseline, never the product
    from tests.configs import brownian

    ora.set_threads(threads)
    B_f = min(cfg["B"], 2 * threads)
    B_b = min(cfg["B"], threads)
    X = brownian(seed, max(B_f, B_b), cfg["L"], cfg["d"]).astype(cfg["dtype"])
    g = np.random.default_rng(seed + 100).standard_normal((B_b, len(ws)))
    ora.forward(X[:1, :3], ws.codes, ws.lengths, cfg["d"])  # load / warm the library
    t0 = time.perf_counter()
    ora.forward(X[:B_f], ws.codes, ws.lengths, cfg["d"])
    t_f = time.perf_counter() - t0
    t0 = time.perf_counter()
    ora.backward(X[:B_b], ws.codes, ws.lengths, cfg["d"], g)
    t_b = time.perf_counter() - t0
    return 1.0 / (t_f / B_f + t_b / B_b), B_f / t_f, t_f, t_b, B_f, B_b


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone times the CPU reference; no process group is formed
    import paper_2602_24066_b200 as sk
    from tests.configs import build_wordset

    cfg = workload(args.config, args.precision)
    ws = build_wordset(args.config, sk)
    threads = cpu_threads()
    for _ in range(args.warmup):
        cpu_sample(args.config, cfg, ws, threads)
    tf = tb = 0.0
    nf = nb = 0
    for _ in range(args.steps):
        _, _, t_f, t_b, B_f, B_b = cpu_sample(args.config, cfg, ws, threads)
        tf += t_f
        tb += t_b
        nf, nb = B_f, B_b
    value = 1.0 / ((tf / args.steps) / nf + (tb / args.steps) / nb)
    dt = "f64" if cfg["dtype"] == np.float64 else "f32"
    sample = (f"per step: forward of {nf} paths ({dt}) + backward of {nb} paths (f64, the reference backward "
              f"contract) of {args.config}; full length L={cfg['L']}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * (tf + tb) / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dt,
        "data": "synthetic Brownian paths (tests/configs.py brownian)",
        "config": {"workload": describe(args.config, cfg, ws), "global_batch": cfg["B"], "length": cfg["L"],
                   "d": cfg["d"], "W": len(ws), "parallelism": "host threads (rank 0 only)"},
        "fwd": {"value": nf * args.steps / tf, "unit": "paths/s"},
        "cpu_baseline": {"value": value, "unit": "paths/s", "cores": threads, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -- GPU arm --------------------------------------------------------------------------------


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2602_24066_b200 as sk
    from paper_2602_24066_b200 import _lib
    from tests.configs import build_wordset

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    _lib.set_kernel_policy(args.policy)
    cfg = workload(args.config, args.precision)
    ws = build_wordset(args.config, sk)
    plan = ws.plan(dev)
    from paper_2602_24066_b200.sharding import shard_range

    if args.batch:
        B = args.batch
    elif args.weak:  # weak scaling: every rank runs the config's batch
        B = cfg["B"]
    else:  # one fixed global batch, contiguous balanced shards (sharding.shard_range)
        lo, hi = shard_range(cfg["B"], rank, world)
        B = hi - lo
    L, d = cfg["L"], cfg["d"]
    M = L - 1
    tdt = torch.float64 if cfg["dtype"] == np.float64 else torch.float32
    dts = "fp64" if tdt == torch.float64 else "fp32"
    W = len(ws)
    sl = sum_lengths(ws)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    # synthetic Brownian paths on [0,1], generated on the device (seed per rank)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 * int(args.config[1]) + rank)
    X = torch.zeros((B, L, d), dtype=tdt, device=dev)
    for s in range(0, B, 8192):
        e = min(B, s + 8192)
        inc = torch.randn((e - s, M, d), generator=gen, dtype=tdt, device=dev) / math.sqrt(max(M, 1))
        torch.cumsum(inc, dim=1, out=X[s:e, 1:])
        del inc
    g = torch.randn((B, W), generator=gen, dtype=tdt, device=dev)
    S = torch.empty((B, W), dtype=tdt, device=dev)
    dXo = torch.empty_like(X)
    work = torch.empty(max(plan.workspace_bytes(tdt, B, L, 0), 1), dtype=torch.uint8, device=dev)

    def step():
        plan.forward(X, S, 0, False)
        plan.backward(X, S, 0, False, g, 0, 0, dXo, work=work)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    barrier()

    # L2 policy: a step whose samples, output and upstream fit twice over in L2
    # (126 MB) would re-read them from L2 on the next step, so those workloads
    # write a 256 MB buffer between timed steps, outside the event brackets.
    l2_bytes = 126 << 20
    step_bytes = (X.numel() + S.numel() + g.numel()) * X.element_size()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if step_bytes < 2 * l2_bytes else None
    l2_note = ("flushed: 256 MB written between timed steps outside the CUDA-event brackets "
               "(X+S+g %.3f GB per rank < 2 x L2)" % (step_bytes / 1e9) if flush is not None else
               "no flush: every pass streams inputs larger than L2 (X %.2f GB, S %.2f GB per rank)"
               % (B * L * d * X.element_size() / 1e9, B * W * X.element_size() / 1e9))

    clocks = ClockSampler(enabled=(local == 0))
    _lib.timing_enable(True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * args.steps)]
    n0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize()
    clocks.mark(True)
    for k in range(args.steps):
        if flush is not None:
            flush.fill_(k & 0xFF)
        ev[3 * k].record()
        plan.forward(X, S, 0, False)
        ev[3 * k + 1].record()
        plan.backward(X, S, 0, False, g, 0, 0, dXo, work=work)
        ev[3 * k + 2].record()
    torch.cuda.synchronize()
    clocks.mark(False)
    barrier()
    launches = _lib.launch_count() - n0
    clk = clocks.stop()
    total_ms = sum(ev[3 * k].elapsed_time(ev[3 * k + 2]) for k in range(args.steps))
    fwd_ms = sum(ev[3 * k].elapsed_time(ev[3 * k + 1]) for k in range(args.steps))
    del flush
    kf_ms, kf_n = _lib.timing_read(0)
    kb_ms, kb_n = _lib.timing_read(1)
    _lib.timing_enable(False)
    total_ms = max_over_ranks(total_ms)
    fwd_ms = max_over_ranks(fwd_ms)
    kf_ms = max_over_ranks(kf_ms)
    kb_ms = max_over_ranks(kb_ms)
    paths_step = B * world if (args.weak or args.batch) else cfg["B"]
    ms_per_step = total_ms / args.steps
    value = paths_step / (ms_per_step / 1e3)
    fwd_value = paths_step * args.steps / (fwd_ms / 1e3)

    peaks = load_peaks()
    peak, peak_src = fma_peak_tflops(dts, sms, peaks)
    peak_ub = ubench_peak_tflops(dts)
    tc_peak, tc_src = tf32_peak_tflops(peaks)
    f_fwd_path = 2.0 * M * sl  # one multiply-add per (word, split)
    f_bwd_path = 3.0 * f_fwd_path
    # the least FMA work a Horner evaluation must execute: one FMA per shared (node, target
    # length) pair per step; the backward needs at least 3 such sweeps
    min_fwd_path = 2.0 * M * plan.step_fmas
    min_bwd_path = 3.0 * min_fwd_path
    tc_fwd = (plan.kernel_kind == 1 and cfg.get("kind") == "truncated" and (d, cfg.get("depth")) == (16, 4)
              and tdt == torch.float32 and os.environ.get("SIGB_TRUNC_TC", "1") != "0")

    def roof(kname, flop_path, min_path, k_ms, k_n, bytes_path):
        if k_n == 0 or k_ms <= 0:
            return None
        sec = k_ms / 1e3
        achieved = flop_path * B * args.steps / sec / 1e12  # per rank, per launch average
        ckey = args.config + ("_fp64" if args.precision == "fp64" else "")  # ncu captures are per dtype
        tr, src = ncu_traffic(kname, ckey)
        per_launch_paths = B * args.steps / k_n
        r = {"bound": "fma", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
             "frac": achieved / peak, "frac_alg": achieved / peak,
             "frac_min_work": min_path * B * args.steps / sec / 1e12 / peak,
             "traffic": None if tr is None else tr * per_launch_paths,
             "algorithmic_bytes": bytes_path * per_launch_paths, "flop_per_launch": flop_path * per_launch_paths,
             "hbm_frac": bytes_path * B * args.steps / sec / 1e9 / float(peaks.get("hbm_gbs", 6456.8)),
             "launch_ms": k_ms / k_n, "launches": k_n, "peak_source": peak_src, "peak_ubench": peak_ub,
             "traffic_source": src, "ncu_exec": ncu_exec(kname, ckey)}
        if kname == "trunc_pq_backward_kernel":
            # both leaf sums on the tensor pipe: D1 = Lambda.dX (over z) and D2 = Lambda^T.dX (over y), each
            # parents x d letters per path-step, 3 fp16 passes (hi.hi + lo.hi + hi.lo), 2 flop per MAC
            leaf_parents = int((np.asarray(ws.lengths) == cfg["depth"] - 1).sum())
            tc_flop = 2 * 3 * 2 * leaf_parents * d * M * B * args.steps / sec / 1e12
            f16_peak = float(peaks.get("bf16_tflops", 2250.0))
            r["tensor"] = {"achieved": tc_flop, "peak": f16_peak, "unit": "TFLOP/s", "frac": tc_flop / f16_peak,
                           "peak_source": "MEASURED_PEAKS.json bf16_tflops (kind::f16 runs at the bf16 rate)",
                           "note": "scaled 3-pass fp16 leaf products on tcgen05 (csrc/sigb_trunc_pq.cuh)"}
        if kname == "trunc_tc_forward_kernel":
            # leaf level on the tensor pipe: 3xTF32 (3 MMAs) x parents x d letters x 2 flop per path-step
            leaf_parents = int((np.asarray(ws.lengths) == cfg["depth"] - 1).sum())
            tc_flop = 3 * 2 * leaf_parents * d * M * B * args.steps / sec / 1e12
            ffma_path = min_fwd_path - 2.0 * M * leaf_parents * d
            t_ffma = ffma_path * B * args.steps / (peak * 1e12)
            t_tc = 3 * 2 * leaf_parents * d * M * B * args.steps / (tc_peak * 1e12)
            r["tensor"] = {"achieved": tc_flop, "peak": tc_peak, "unit": "TFLOP/s", "frac": tc_flop / tc_peak,
                           "peak_source": tc_src,
                           "note": "3xTF32 leaf update (hi.hi + hi.lo + lo.hi) executed on tcgen05"}
            r["frac_combined"] = max(t_ffma, t_tc) / sec
            r["combined_note"] = ("bound = max(non-leaf shared-Horner FFMA / FFMA peak, 3xTF32 leaf MMA flop / "
                                  "tf32 peak); frac_combined = that bound / measured time")
        return r

    s_el = 8 if tdt == torch.float64 else 4
    bytes_fwd = (L * d + W) * s_el
    bytes_bwd = (2 * L * d + 2 * W) * s_el
    prefix = {1: "trunc_", 2: "frag_"}.get(plan.kernel_kind, "")
    kb_name, kf_name = prefix + "backward_kernel", prefix + "forward_kernel"
    if plan.kernel_kind == 4:
        kb_name, kf_name = "sigjit_bwd", "sigjit_fwd"
    if tc_fwd:
        kf_name = "trunc_tc_forward_kernel"  # leaf level on the tensor cores (csrc/sigb_trunc_tc.cuh)
    pq_bwd = (plan.kernel_kind == 1 and cfg.get("kind") == "truncated" and tdt == torch.float32
              and (d, cfg.get("depth")) in ((16, 4), (8, 5)) and os.environ.get("SIGB_TRUNC_TC_BWD", "2") == "2")
    if pq_bwd:
        kb_name = "trunc_pq_backward_kernel"  # both leaf sums on the tensor cores (csrc/sigb_trunc_pq.cuh)
    roof_b = roof(kb_name, f_bwd_path, min_bwd_path, kb_ms, kb_n, bytes_bwd)
    roof_f = roof(kf_name, f_fwd_path, min_fwd_path, kf_ms, kf_n, bytes_fwd)
    dominant = roof_b if (roof_b and kb_ms >= kf_ms) else roof_f

    del work
    # -- optional all-gather of S (kept out of the headline) -----------
    gather = None
    if args.gather and world > 1:
        Bg = min(B, max(1, (4 << 30) // (W * s_el * world)))
        src = S[:Bg].contiguous()
        dst = torch.empty((Bg * world, W), dtype=tdt, device=dev)
        for _ in range(2):
            dist.all_gather_into_tensor(dst, src)
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            dist.all_gather_into_tensor(dst, src)
        b.record()
        torch.cuda.synchronize()
        gms = max_over_ranks(a.elapsed_time(b) / 3)
        gather = {"paths_per_rank": Bg, "ms": gms, "bytes_received_per_rank": Bg * W * s_el * (world - 1),
                  "GBps_per_rank": Bg * W * s_el * (world - 1) / (gms / 1e3) / 1e9}
        del src, dst

    # -- end to end: public API, host buffers --------------------------------------------
    e2e = e2e_fwd = e2e_dropin = None
    if not args.no_e2e:
        del S, g, dXo
        torch.cuda.empty_cache()
        Xh = X.cpu().pin_memory()
        del X
        torch.cuda.empty_cache()
        readout = torch.randn((W,), generator=gen, dtype=tdt, device=dev)
        # A step is the whole batch as `split` sub-batches pushed through a copy /
        # compute / copy pipeline, as a training loop would stream micro-batches:
        # sub-batch u+1's H2D (own stream) and u-1's D2H (own stream) overlap u's
        # compute.  Every sub-batch's inputs go in and its dL/dX and loss come out
        # inside the timed region; only the first H2D and the last D2H of the run
        # are exposed.
        # sub-batches of >= 2 ms of device work each (from this run's timed step): a sub-batch's
        # launches and autograd bookkeeping cost ~0.1-0.3 ms, which smaller pieces cannot hide;
        # at most --e2e-split of them
        split = max(1, min(args.e2e_split, B // 32, int(ms_per_step / 2.0)))
        bounds_u = [(B * i // split, B * (i + 1) // split) for i in range(split)]
        ub = max(hi - lo for lo, hi in bounds_u)
        dXh = torch.empty_like(Xh).pin_memory()
        lossh = torch.empty((args.steps + 4, split), dtype=tdt).pin_memory()
        Xbuf = [torch.empty((ub,) + tuple(Xh.shape[1:]), dtype=tdt, device=dev) for _ in range(2)]
        main = torch.cuda.current_stream(dev)
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ready = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]
        fin = torch.cuda.Event()

        def e2e_run(nsteps, start_ev=None):
            units = [(k, i) for k in range(nsteps) for i in range(split)]

            def issue(u):
                lo, hi = bounds_u[units[u][1]]
                with torch.cuda.stream(h2d):
                    if start_ev is not None and u == 0:
                        h2d.wait_event(start_ev)
                    if u >= 2:
                        h2d.wait_event(freed[u % 2])  # unit u-2 no longer reads this buffer
                    Xbuf[u % 2][: hi - lo].copy_(Xh[lo:hi], non_blocking=True)
                    ready[u % 2].record(h2d)

            issue(0)
            for u, (k, i) in enumerate(units):
                lo, hi = bounds_u[i]
                if u + 1 < len(units):
                    issue(u + 1)
                main.wait_event(ready[u % 2])
                Xd = Xbuf[u % 2][: hi - lo].detach().requires_grad_(True)
                Sd = sk.signature(Xd, ws)
                loss = (Sd @ readout).sum()
                loss.backward()
                grad = Xd.grad
                freed[u % 2].record(main)
                with torch.cuda.stream(d2h):
                    d2h.wait_event(freed[u % 2])
                    dXh[lo:hi].copy_(grad, non_blocking=True)
                    lossh[k, i].copy_(loss.detach(), non_blocking=True)
                grad.record_stream(d2h)
                loss.record_stream(d2h)
                del Sd, loss, grad, Xd
            fin.record(d2h)
            main.wait_event(fin)

        e2e_run(max(1, min(args.warmup, 2)))
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        e2e_run(args.steps, start_ev=a)
        b.record()
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(a.elapsed_time(b)) / args.steps
        e2e = {"value": paths_step / (ems / 1e3), "unit": "paths/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(Xh.numel() * Xh.element_size()),
               "d2h_bytes_per_step": int(dXh.numel() * dXh.element_size() + split * lossh.element_size()),
               "api": "paper_2602_24066_b200.signature (autograd) on pinned host paths; loss = (S @ r).sum(); "
                      "dL/dX and loss copied back; the batch streams as %d sub-batches with H2D / D2H on their "
                      "own streams overlapping the neighbouring sub-batches' compute" % split}
        # forward through the numpy drop-in (signature_forward: host array in, host array out)
        # host result buffers are pinned: keep them to ~2 GB per rank (8 ranks share one host)
        Bn = min(B, max(1, (2 << 30) // (W * s_el)))
        Xn = Xh[:Bn].numpy()
        del Xh, dXh, Xbuf
        torch.cuda.empty_cache()
        sk.signature_forward(Xn, ws)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        reps = max(1, min(args.steps, 3))
        for _ in range(reps):
            sk.signature_forward(Xn, ws)
        torch.cuda.synchronize()
        fms = max_over_ranks((time.perf_counter() - t0) * 1e3 / reps)
        e2e_fwd = {"value": Bn * world / (fms / 1e3), "unit": "paths/s", "ms_per_step": fms,
                   "paths_per_rank": Bn, "h2d_bytes_per_step": int(Xn.nbytes), "d2h_bytes_per_step": Bn * W * s_el,
                   "api": "signature_forward(numpy) -> CoefficientBatch(numpy); host-synchronous wall clock"}
        # the reference's drop-in pair on host arrays: signature_forward + signature_backward, the backward
        # in float64 as its contract requires (backward.py:166-167); host upstream of the same shape
        Bd = min(Bn, max(1, (1 << 30) // (W * 8)))
        Xd = Xn[:Bd]
        gd = np.random.default_rng(7).standard_normal((Bd, W))
        sk.signature_forward(Xd, ws)  # full-size warm-up: the pinned host blocks get cached
        sk.signature_backward(Xd, ws, gd)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            sk.signature_forward(Xd, ws)
            sk.signature_backward(Xd, ws, gd)
        dms = max_over_ranks((time.perf_counter() - t0) * 1e3 / reps)
        e2e_dropin = {"value": Bd * world / (dms / 1e3), "unit": "paths/s", "ms_per_step": dms, "paths_per_rank": Bd,
                      "h2d_bytes_per_step": int(Xd.nbytes + 8 * Bd * W + 8 * Xd.size),
                      "d2h_bytes_per_step": int(Bd * W * s_el + 8 * Bd * (L - 1) * d + 8 * Xd.size),
                      "api": "signature_forward(numpy) + signature_backward(numpy, float64 upstream) -> GradBatch; "
                             "the backward always computes in float64 (the reference contract)"}

    # -- CPU baseline (rank 0, N = 1 only) -------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        v, vf, t_f, t_b, B_f, B_b = cpu_sample(args.config, cfg, ws, threads)
        cpu = {"value": v, "unit": "paths/s", "cores": threads, "kind": "port", "fwd_value": vf, "cpu_model": cpu_model(),
               "sample": f"oracle port (oracle/sig_oracle.c, OpenMP) of the reference numba kernels: forward of "
                         f"{B_f} paths ({'f64' if tdt == torch.float64 else 'f32'}) in {t_f:.2f} s + backward of "
                         f"{B_b} paths (f64, reference contract) in {t_b:.2f} s, full L={L}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if (args.weak or args.batch) else "strong", "vs_baseline": None, "dtype": dts.replace("fp", "f"),
            "data": "synthetic Brownian paths on [0,1] (dX ~ N(0, 1/M)), generated on device per rank; "
                    "dense N(0,1) upstream",
            "config": {"workload": describe(args.config, cfg, ws), "per_rank_batch": B, "global_batch": paths_step,
                       "length": L, "d": d, "W": W, "sum_word_len": sl,
                       "parallelism": f"dp{world}: batch-sharded, no collective in fwd/bwd",
                       "l2": l2_note,
                       "kernels": "%s: fwd %s, bwd %s" % (
                           {1: "truncated", 2: "fragment", 4: "word-set generated (NVRTC)"}.get(
                               plan.kernel_kind, "level-synchronous trie"),
                           kf_name, kb_name)},
            "fwd": {"value": fwd_value, "unit": "paths/s", "ms_per_step": fwd_ms / args.steps},
            "roofline": dominant, "roofline_fwd": roof_f if dominant is not roof_f else roof_b,
            "cpu_baseline": cpu, "e2e": e2e, "e2e_fwd": e2e_fwd, "e2e_dropin_fwd_bwd": e2e_dropin, "gather": gather,
            "gpu_launches": launches, "clocks": clk,
        }
        if "paper_ms" in cfg:  # pathsig's own H200 training time for this row (context, not a baseline)
            line["paper_context"] = {"row": cfg["paper_row"], "pathsig_h200_ms": cfg["paper_ms"],
                                     "pathsig_h200_paths_per_s": cfg["B"] / (cfg["paper_ms"] / 1e3),
                                     "source": "/root/reference/PAPER.md:429-449 (training time, fwd+bwd)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def self_launch(args, argv) -> int:
    """`--gpus N` outside torchrun: re-run this script as N ranks under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1), the launch the driver itself uses."""
    import socket

    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)
    return subprocess.run(cmd, cwd=ROOT).returncode


def main(argv=None) -> None:
    argv = sys.argv[1:] if argv is None else list(argv)
    args = parse_args(argv)
    if args.impl == "reference":
        run_reference(args)  # rank 0 alone; no process group
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args, argv))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and int(os.environ.get("RANK", "0")) == 0:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; timing {world} rank(s)\n")
    run_ours(args)


if __name__ == "__main__":
    main()
