"""Benchmark of the LARS data-parallel step (ResNet-50 parameter set).

One "step" = one pass of the hot path over one batch of synthetic gradients:
at N=1 the fused lars_step kernel; at N>1 reduce-scatter -> partial norms ->
norm all-reduce -> update -> all-gather (cluster.DataParallelLars), with
inputs resident in HBM.  `value` is whole-job algorithmic throughput,
20 B/param (fp32 read w, g, m; write w, m) x params / step time, in GB/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet50|alexnet_bn|sweep:<N>:<L>]

Under torchrun (N>1) every rank runs; rank 0 prints one JSON line.  Timing:
CUDA events on the launching stream around every step, L2 flushed between
steps (1 GiB write, untimed), barrier + synchronize around the timed region,
max over ranks.  Extras on the line: `roofline` (kernel time vs the measured
HBM peak; DRAM bytes of one launch measured in-run with ncu), `e2e` (pinned
host gradient in, lambdas out, through DataParallelLars), `e2e_host_paramset`
(N=1: the literal reference call, optim.apply_update on a host fp64
ParamSet), `cpu_baseline` (the reference's apply_update on this host) and
`resnet50_train` (img/s at global batch 32K).  `--impl reference` times the
unmodified reference (`batchlab`, pip-installed into baseline/_ref) through
its own API on the same workload, rank 0 only; the oracle port stands in if
baseline/_ref is missing.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

BYTES_PER_PARAM = 20  # read w, g, m + write w, m (fp32)
PEAKS_FILE = os.path.join(HERE, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
GLOBAL_BATCH = 32768


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the in-run ncu capture of the kernel's DRAM bytes")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--host-e2e-steps", type=int, default=10,
                    help="N=1: also time optim.apply_update on a host fp64 ParamSet (0: skip)")
    ap.add_argument("--train-steps", type=int, default=5,
                    help="also time ResNet-50 training steps at global batch 32K (0: skip)")
    ap.add_argument("--backend", default="auto", choices=["auto", "nccl", "p2p", "p2p-stream"],
                    help="N>1: NCCL collectives around the split kernels, or the peer-memory fused kernel (p2p)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def workload_config(name, layout, n_gpus):
    from paper_1709_05011_b200 import layouts
    return {
        "workload": f"{name} parameter set, LARS DP step (RS->LARS->AG at N>1)",
        "params": layouts.total_params(layout),
        "layers": len(layout),
        "global_batch": GLOBAL_BATCH,
        "state": "fp32 w/g/m, fp64 norms and trust ratios",
        "l2": "flushed between timed steps (1 GiB write + 256 MiB read, untimed)",
        "rank_alignment": "N>1: a device-side cross-rank barrier after each untimed flush, before the step's start event",
        "parallelism": f"dp{n_gpus}" + ("-sharded (ZeRO-1 momentum)" if n_gpus > 1 else ""),
    }


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, local_rank, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1709_05011_b200 import layouts, optim
    from paper_1709_05011_b200.cluster import DataParallelLars
    from paper_1709_05011_b200.flat import FlatParamSet

    layout = layouts.get(args.workload)
    n_params = layouts.total_params(layout)
    params = FlatParamSet(layout, dev, world_size=world, rank=rank,
                          symmetric=(world > 1 and args.backend != "nccl"))
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)  # same weights on every rank
    for grp in params:
        if grp.category == "norm-scale":
            grp.param.fill_(1.0)
        elif grp.category == "weight":
            grp.param.uniform_(-0.05, 0.05, generator=gen)
    gen.manual_seed(5678 + rank)  # per-rank local gradient (sum convention)
    for grp in params:
        grp.grad.normal_(0.0, 1e-3 * GLOBAL_BATCH / world, generator=gen)
    params.invalidate_norm_cache()
    # config 4 recipe: linear scaling 0.2 @ 256 -> 25.6 @ 32K, 5 warmup epochs, poly 2
    n_images = 1_281_167
    hp = optim.HyperParams(base_lr=optim.linear_scaled_lr(0.2, 256, GLOBAL_BATCH), epochs=90,
                           batch_size=GLOBAL_BATCH, momentum=0.9, weight_decay=5e-4,
                           poly_power=2.0, warmup_epochs=5, lars_enabled=True, lars_trust=1e-3)
    ipe = n_images // GLOBAL_BATCH
    st = optim.ScheduleState(optim.max_iterations(90, n_images, GLOBAL_BATCH), ipe)
    dp = DataParallelLars(params, backend=args.backend if world > 1 else "auto")
    grad_scale = 1.0 / GLOBAL_BATCH
    flush_buf = torch.empty(1 << 28, dtype=torch.float32, device=dev)  # 1 GiB
    clean_buf = torch.ones(1 << 26, dtype=torch.float32, device=dev)   # 256 MiB
    stream = torch.cuda.current_stream()

    class _Flush:
        """Evict L2 between steps: write 1 GiB, then read 256 MiB so the L2
        holds clean unrelated lines (no write-backs billed to the next step)."""

        def zero_(self):
            flush_buf.zero_()
            clean_buf.sum()

    flush = _Flush()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    # warm-up (also makes the momentum nonzero and the norm carry valid).  The
    # first step is checked: if a peer-memory kernel's cross-rank barrier
    # timed out (LARS_STATUS_RANK_TIMEOUT -> ProtocolError on every rank), the
    # line is measured on the NCCL backend instead and says so
    fallback = None
    from paper_1709_05011_b200.errors import DivergenceError, ProtocolError
    try:
        flush.zero_()
        dp.step(hp, st, grad_scale=grad_scale, check=True)
    except DivergenceError:
        pass  # synthetic gradients: reported in last_step, not fatal for timing
    except ProtocolError as e:
        if world == 1 or dp.backend == "nccl":
            raise
        fallback = f"{dp.backend} backend failed its first step ({e}); measured on nccl"
        if rank == 0:
            print(f"# {fallback}", file=sys.stderr)
        dp = DataParallelLars(params, backend="nccl")
        params.invalidate_norm_cache()
        dp.step(hp, st, grad_scale=grad_scale)
    for _ in range(max(args.warmup, 3) - 1):
        flush.zero_()
        dp.step(hp, st, grad_scale=grad_scale)
    graphed = None
    if not args.no_graph:
        try:
            graphed = dp.capture(hp, st, grad_scale=grad_scale)
            flush.zero_()
            graphed.replay()
        except Exception as e:  # capture unsupported -> eager launches
            graphed = None
            if rank == 0:
                print(f"# graph capture unavailable: {e!r}", file=sys.stderr)
    torch.cuda.synchronize()

    # ---- timed region: K steps ----
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)  # let nvidia-smi attach before the timed region
    barrier()
    evs = []
    for _ in range(args.steps):
        flush.zero_()
        dp.align(hp)  # N>1: ranks leave the flush together (device barrier, untimed)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if graphed is not None:
            graphed.replay()
        else:
            dp.step(hp, st, grad_scale=grad_scale)
        b.record(stream)
        evs.append((a, b))
    barrier()
    # the timed region is milliseconds long: keep the identical step loop
    # running (untimed) for >=1.5 s so the 100 ms clock samples see the load.
    # The count is fixed up front and identical on every rank (a step is a
    # cross-rank barrier at N>1: a time-based loop could run a different
    # number of steps per rank)
    per_step = torch.tensor([max(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(per_step, op=dist.ReduceOp.MAX)
    step_wall_ms = float(per_step.item()) + 0.05  # + the untimed flush
    n_soak = min(20000, max(20, int(1500.0 / step_wall_ms)))
    for i in range(n_soak):
        if st.iteration > st.max_iterations - 100:
            st.iteration = 200  # stay inside the schedule while soaking
        flush.zero_()
        if graphed is not None:
            graphed.replay()
        else:
            dp.step(hp, st, grad_scale=grad_scale)
        if i % 20 == 19:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)

    # ---- kernel-only timing (the roofline denominator's kernel) ----
    phases = {}
    kern_ms = []
    for _ in range(args.steps):
        flush.zero_()
        dp.align(hp)
        timers = []
        dp.step(hp, st, grad_scale=grad_scale, timers=timers)
        for (n0, e0), (n1, e1) in zip(timers, timers[1:]):
            phases.setdefault(n1, []).append((e0, e1))
    torch.cuda.synchronize()
    phase_ms = {k: statistics.median([a.elapsed_time(b) for a, b in v]) for k, v in phases.items()}
    if world == 1 or "lars_step_peer" in phase_ms or "lars_step_peer_stream" in phase_ms:
        # the step is one kernel launch: its duration is the timed region's
        # per-step event time (median); the eager re-measurement above stays
        # in phases_us
        kern_ms = statistics.median(step_ms)
        kern_src = "timed region: CUDA events around each step (one kernel launch per step)"
    else:
        kern_ms = phase_ms["partial_norms"] + phase_ms["update"]
        kern_src = "eager re-run: CUDA events around partial_norms + update (median)"

    # ---- end to end through the public API with host buffers ----
    host_grad = params.flat_grad.detach().cpu().pin_memory()
    e2e_ms = []
    for _ in range(args.e2e_steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        barrier()
        a.record(stream)
        params.set_grads(host_grad)                            # H2D, pinned
        lams = dp.step(hp, st, grad_scale=grad_scale)          # the DP step
        lam_host = dict(lams)                                  # D2H of the result
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    assert len(lam_host) == len(layout)

    # max over ranks
    vals = torch.tensor([total_ms, kern_ms, statistics.median(e2e_ms)], dtype=torch.float64,
                        device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        ph = torch.tensor([phase_ms[k] for k in sorted(phase_ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(ph, op=dist.ReduceOp.MAX)
        phase_ms = dict(zip(sorted(phase_ms), ph.tolist()))
    total_ms, kern_ms, e2e_med = vals.tolist()

    info = optim.step_info(params)
    scale_defs = None
    if world > 1:
        scale_defs = scaling_legs(args, layout, params, hp, st, grad_scale, flush, world,
                                  total_ms / args.steps * 1e3, kern_ms * 1e3, dev)
    local = params.shard_numel
    n_padded = params.padded_numel
    backend = dp.backend
    use_graph = graphed is not None
    train = None
    if args.train_steps > 0 and args.workload == "resnet50":
        del dp, params, flush_buf, clean_buf, graphed
        torch.cuda.empty_cache()
        train = resnet50_train(args, world, rank, local_rank, dev)
        if world > 1 and "error" not in train and str(train.get("dp_backend")).startswith("p2p"):
            train["exposed_step_us"] = exposed_step(world, dev)

    def finish():
        # NCCL work captured in a CUDA graph can make process-group teardown
        # hang: synchronise every rank, then leave without teardown
        if world > 1:
            dist.barrier(device_ids=[local_rank])
            torch.cuda.synchronize()
            sys.stdout.flush()
            sys.stderr.flush()
            os._exit(0)

    if rank != 0:
        finish()
        return

    peak, peak_kind = hbm_peak()
    ms_per_step = total_ms / args.steps
    value = BYTES_PER_PARAM * n_params / (ms_per_step * 1e-3) / 1e9

    achieved = BYTES_PER_PARAM * local / (kern_ms * 1e-3) / 1e9
    # DRAM bytes of one launch of THIS build, measured in-run with ncu on the
    # same workload (byte counts only; N=1: the cross-rank peer kernel cannot
    # be replayed by a single-process ncu)
    traffic = {"error": "not captured (--no-traffic)"} if args.no_traffic else (
        {"error": "N>1: cross-rank kernel"} if world > 1 else None)
    if traffic is None:
        sys.path.insert(0, os.path.join(HERE, "tools"))
        import traffic_capture
        traffic = traffic_capture.capture(args.workload)
    t_read, t_write = traffic.get("read"), traffic.get("write")
    alg_write = 8 * local  # w and m written back, fp32
    line = {
        "metric": "LARS step HBM GB/s (algorithmic 20 B/param; % of roofline in 'roofline')",
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (random-init weights, N(0,sigma) gradients)",
        "config": workload_config(args.workload, layout, world),
        "graph": use_graph,
        "backend": backend,
        "backend_fallback": fallback,
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 2),
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": (t_read + t_write) if t_read is not None else None,
            "traffic_read": t_read,
            "traffic_write": t_write,
            "traffic_source": ("ncu dram__bytes_read/write.sum, one launch of this build "
                               "(tools/traffic_capture.py, run by this bench)")
                              if t_read is not None else traffic.get("error"),
            # w/m lines still dirty in L2 when the kernel ends are written back
            # after it (in the bench: during the untimed flush); billing them at
            # peak HBM bandwidth to the step:
            "frac_writeback_billed": round(
                BYTES_PER_PARAM * local / (kern_ms * 1e-3 + max(0, alg_write - t_write) / (peak * 1e9))
                / 1e9 / peak, 4) if t_write is not None else None,
            "kernel_us": round(kern_ms * 1e3, 2),
            "kernel_timing": kern_src,
            "bytes_per_launch": BYTES_PER_PARAM * local,
            # lambda needs both norms before any update: g is read twice
            # (24 B/param unless the re-read hits L2) -- DESIGN.md section 3
            "two_pass_bound_us": round(24 * local / (peak * 1e9) * 1e6, 2),
            "frac_of_two_pass_bound": round(24 * local / (peak * 1e9) / (kern_ms * 1e-3), 4),
        },
        "phases_us": {k: round(v * 1e3, 2) for k, v in phase_ms.items()},
        "e2e": {
            "value": round(BYTES_PER_PARAM * n_params / (e2e_med * 1e-3) / 1e9, 2),
            "unit": "GB/s",
            "ms_per_step": round(e2e_med, 4),
            "h2d_bytes_per_step": 4 * n_padded * world,
            "d2h_bytes_per_step": 8 * len(layout) * world,
            "path": "FlatParamSet.set_grads(pinned host) + DataParallelLars.step + dict(lambdas)",
        },
        "gpu_launches": args.steps * (2 if backend == "nccl" else 1),
        "clocks": clocks,
        "last_step": {"lr": info[0], "iteration": info[1],
                      "nonfinite_layer": None if info[2] == 2**31 - 1 else info[2]},
    }
    if train is not None:
        line["resnet50_train"] = train
    if scale_defs is not None:
        line["scaling_defs"] = scale_defs
    if world > 1:
        # NVLink byte counters: NVML reports the NVLINK_THROUGHPUT / COUNT_XMIT
        # fields as not supported on these (virtualised) boxes and nvidia-smi
        # shows N/A (profiles/r02_nvlink_counters.txt), so link bytes are the
        # algorithmic ones in scaling_defs
        line["nvlink_counters"] = {"available": False,
                                   "why": "NVML NVLINK_THROUGHPUT_* fields: NOT_SUPPORTED on this box"}
        nbytes = 4 * n_padded
        for k in ("reduce_scatter", "all_gather"):
            if k in phase_ms:
                line.setdefault("busbw_gbs", {})[k] = round(
                    (world - 1) / world * nbytes / (phase_ms[k] * 1e-3) / 1e9, 1)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(layout, seconds=12.0)
    if world == 1 and args.host_e2e_steps > 0:
        line["e2e_host_paramset"] = e2e_host_paramset(
            layout, args.host_e2e_steps, (line.get("cpu_baseline") or {}).get("ms_per_step"))
    print(json.dumps(line), flush=True)
    finish()


def _fused_kernel_us(params, hp, st, grad_scale, steps, flush):
    """Median time of the single-GPU fused lars_step kernel over this rank's
    shard of `params` (no communication): the kernel-only strong-scaling leg."""
    import torch
    from paper_1709_05011_b200 import _native as nat
    from paper_1709_05011_b200.flat import _ptr
    from paper_1709_05011_b200.optim import native_hparams
    eng = params.engine()
    key = frozenset(hp.lars_skip_categories)
    plan, ws = eng.plan(key)
    lib = nat.load()
    stream = torch.cuda.current_stream()
    w, g, m = params.param_shard, params.grad_shard_of_full, params.momentum
    ts = []
    for i in range(steps + 3):
        flags = nat.LARS_STEP_USE_WCARRY if i > 0 else 0
        h = native_hparams(hp, st, lr=0.01, grad_scale=grad_scale, flags=flags)
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        nat.check(lib.lars_step(plan.handle, _ptr(w), _ptr(g), _ptr(m), nat.ctypes.byref(h),
                                _ptr(eng.d_iter), _ptr(eng.d_sumsq), _ptr(eng.d_lambda),
                                _ptr(eng.d_info), _ptr(ws), stream.cuda_stream))
        b.record(stream)
        if i >= 3:
            ts.append((a, b))
    torch.cuda.synchronize()
    eng.invalidate()
    return statistics.median([a.elapsed_time(b) for a, b in ts]) * 1e3


def scaling_legs(args, layout, params, hp, st, grad_scale, flush, world, step_us, kern_us, dev):
    """SURVEY §8e efficiency definitions at N>1 (max over ranks):
    (1) kernel-only strong scaling E_k = T_fused(N) / (P * T_fused(N/P));
    (2) sharded-step roofline E_s = [2(P-1)/P*4N/900 GB/s + 20N/P/HBM] / T_step."""
    import torch
    import torch.distributed as dist
    from paper_1709_05011_b200.flat import FlatParamSet
    t_shard = torch.tensor([_fused_kernel_us(params, hp, st, grad_scale, 10, flush)],
                           dtype=torch.float64, device=dev)
    dist.all_reduce(t_shard, op=dist.ReduceOp.MAX)
    full = FlatParamSet(layout, dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    for grp in full:
        grp.param.uniform_(-0.05, 0.05, generator=gen)
        grp.grad.normal_(0.0, 1e-3 * GLOBAL_BATCH, generator=gen)
    t1 = _fused_kernel_us(full, hp, st, grad_scale, 10, flush)
    del full
    n = params.padded_numel
    peak, _ = hbm_peak()
    ideal_us = (2 * (world - 1) / world * 4 * n / 900e9 + BYTES_PER_PARAM * n / world / (peak * 1e9)) * 1e6
    link_bytes = 2 * (world - 1) / world * 4 * n
    return {
        "kernel_only_strong_eff": round(t1 / (world * float(t_shard)), 4),
        "t_fused_full_us": round(t1, 2),
        "t_fused_shard_us_max": round(float(t_shard), 2),
        "step_roofline_eff": round(ideal_us / step_us, 4),
        "step_ideal_us": round(ideal_us, 2),
        "nvlink_bytes_per_rank": int(link_bytes),
        "nvlink_gbs_per_direction": round(link_bytes / (kern_us * 1e-6) / 1e9, 1),
        "nvlink_peak_gbs": 900,
    }


def exposed_step(world, dev):
    """Time from the end of backward to the end of the LARS step (one
    micro-batch of 256 per rank), plain p2p step vs the backward-overlapped
    gradient push (tools/overlap_time.py; min over ranks = the rank whose
    backward ends last)."""
    try:
        sys.path.insert(0, os.path.join(HERE, "tools"))
        import overlap_time
        out = {}
        for mode in (False, True):
            _, ex_lo, _ = overlap_time.run(mode, 8, 256)
            out["overlap" if mode else "plain"] = round(ex_lo, 1)
        return out
    except Exception as e:  # report, do not lose the main line
        return {"error": repr(e)[:200]}


def resnet50_train(args, world, rank, local_rank, dev):
    """ResNet-50 img/s at global batch 32K: synthetic ImageNet-shape data,
    random-init weights, micro-batches of 256 accumulated into the flat
    gradient, then the sharded LARS step (paper_1709_05011_b200.train)."""
    import torch
    import torch.distributed as dist
    from paper_1709_05011_b200 import optim
    from paper_1709_05011_b200.train import Trainer, build_model
    try:
        micro = 256
        torch.manual_seed(0)
        torch.backends.cudnn.benchmark = True
        n_images = 1_281_167
        hp = optim.HyperParams(base_lr=optim.linear_scaled_lr(0.2, 256, GLOBAL_BATCH), epochs=90,
                               batch_size=GLOBAL_BATCH, warmup_epochs=5, lars_enabled=True)
        st = optim.ScheduleState(optim.max_iterations(90, n_images, GLOBAL_BATCH),
                                 n_images // GLOBAL_BATCH)
        # p2p backend: gradient buckets pushed during the last backward (§8f1)
        tr = Trainer(build_model("resnet50"), hp, st, GLOBAL_BATCH, micro, dev, args.backend,
                     overlap=True)
        g = torch.Generator(device=dev)
        g.manual_seed(99 + rank)
        x = torch.randn(micro, 3, 224, 224, device=dev, generator=g).to(
            memory_format=torch.channels_last)
        y = torch.randint(0, 1000, (micro,), device=dev, generator=g)
        batches = [(x, y)] * tr.accum
        tr.step(batches)  # one full warm-up step (cudnn autotune, plan, workspace, overlap hooks)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        evs = []
        for _ in range(args.train_steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            tr.step(batches)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        per = torch.tensor([a.elapsed_time(b) for a, b in evs], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(per, op=dist.ReduceOp.MAX)
        per = per.tolist()
        step_ms = statistics.median(per)
        return {"metric": "ResNet-50 img/s at global batch 32768", "value": round(GLOBAL_BATCH / (step_ms * 1e-3), 1),
                "unit": "img/s", "ms_per_step": round(step_ms, 1), "micro_batch": micro,
                "accum_per_gpu": tr.accum, "steps": args.train_steps, "warmup_steps": 1,
                "step_ms_min_med_max": [round(min(per), 1), round(step_ms, 1), round(max(per), 1)],
                "dp_backend": tr.dp.backend,
                "backward_overlap": tr.overlap is not None,
                "precision": "bf16 autocast fwd/bwd, fp32 master weights/grads/momentum",
                "data": "synthetic 224x224x3, 1000 classes, random-init weights",
                "scaling": "strong (global batch fixed at 32768)"}
    except Exception as e:  # report, do not lose the main line
        return {"error": repr(e)[:300]}


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference)
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(HERE, "baseline", "_ref")


def stock_reference():
    """The unmodified reference package `batchlab` (pip-installed from
    /root/reference into baseline/_ref), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "batchlab")):
        return None
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import batchlab.cluster  # noqa: F401
        import batchlab.nn  # noqa: F401
        import batchlab.optim  # noqa: F401
        import batchlab
        return batchlab
    except Exception:
        return None


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _host_arrays(layout, seed=0):
    """Seeded fp64 (w, g, m) per group, the reference's array type."""
    import numpy as np
    rng = np.random.default_rng(seed)
    out = []
    for name, shape, cat in layout:
        n = int(np.prod(shape))
        w = rng.uniform(-0.05, 0.05, n) if cat == "weight" else np.ones(n)
        g = rng.standard_normal(n) * 1e-3
        out.append((name, w.reshape(shape), g.reshape(shape), np.zeros(shape), cat))
    return out


def _oracle_groups(layout, seed=0):
    from oracle import lars_oracle as orc
    return [orc.Group(n, w, g, m, c) for n, w, g, m, c in _host_arrays(layout, seed)]


def _stock_paramset(ref, layout, seed=0):
    return ref.nn.ParamSet(ref.nn.ParamGroup(n, w, g, m, c) for n, w, g, m, c in _host_arrays(layout, seed))


def _recipe_kw():
    # config 4 recipe (optim.py:25-36 fields)
    return dict(base_lr=25.6, epochs=90, batch_size=GLOBAL_BATCH, momentum=0.9, weight_decay=5e-4,
                poly_power=2.0, warmup_epochs=5, lars_enabled=True, lars_trust=1e-3)


class _HP:
    """Duck-typed HyperParams for the oracle port."""

    def __init__(self):
        from oracle import lars_oracle as orc
        for k, v in _recipe_kw().items():
            setattr(self, k, v)
        self.lars_skip_categories = orc.DEFAULT_LARS_SKIP


def _timed(run, seconds, min_calls=3):
    run()
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < min_calls:
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    return times


def cpu_baseline(layout, seconds):
    """Time the reference's apply_update (optim.py:117-134) on the same
    parameter set on this host: the stock `batchlab` from baseline/_ref when
    it is installed (kind "reference"), else the oracle's restatement
    (kind "port").  One warm call, then calls until ~`seconds` elapse."""
    from paper_1709_05011_b200 import layouts
    ref = stock_reference()
    if ref is not None:
        params = _stock_paramset(ref, layout)
        hp = ref.optim.HyperParams(**_recipe_kw())
        run = lambda: ref.optim.apply_update(params, hp, 0.1)  # noqa: E731
        kind, what = "reference", "batchlab.optim.apply_update (stock, baseline/_ref)"
    else:
        from oracle import lars_oracle as orc
        groups = _oracle_groups(layout)
        hp = _HP()
        run = lambda: orc.apply_update(groups, hp, 0.1)  # noqa: E731
        kind, what = "port", "oracle apply_update (restatement)"
    times = _timed(run, seconds)
    n = layouts.total_params(layout)
    med = statistics.median(times)
    return {"value": round(BYTES_PER_PARAM * n / med / 1e9, 4), "unit": "GB/s", "cores": 1,
            "kind": kind, "ms_per_step": round(med * 1e3, 2),
            "sample": f"{len(times)} x {what} on the full {len(layout)}-group, {n}-param set "
            f"(fp64 numpy, single-threaded numpy elementwise; OPENBLAS_NUM_THREADS="
            f"{os.environ.get('OPENBLAS_NUM_THREADS', 'unset')}), median {med * 1e3:.1f} ms",
            "cpu_model": cpu_model(), "host_threads": os.cpu_count()}


def e2e_host_paramset(layout, steps, cpu_ms):
    """The literal drop-in: optim.apply_update on a reference-style ParamSet
    of caller-owned fp64 numpy arrays (the stock batchlab.nn.ParamSet when
    installed), w / g / m DMA'd in from the caller's memory and w / m
    written back in place every call (hostset.py), lambdas returned as a
    dict.  Wall clock per call (it ends with a synchronize)."""
    from paper_1709_05011_b200 import layouts, optim
    ref = stock_reference()
    if ref is not None:
        params = _stock_paramset(ref, layout)
        kind = "batchlab.nn.ParamSet (stock)"
    else:
        params = _oracle_groups(layout)
        kind = "oracle Group list"
    hp = optim.HyperParams(**_recipe_kw())
    for _ in range(3):
        optim.apply_update(params, hp, 0.1, iteration=0)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        lams = optim.apply_update(params, hp, 0.1, iteration=0)
        times.append(time.perf_counter() - t0)
    assert len(lams) == len(layout)
    n = layouts.total_params(layout)
    med = statistics.median(times)
    out = {"value": round(BYTES_PER_PARAM * n / med / 1e9, 3), "unit": "GB/s",
           "ms_per_step": round(med * 1e3, 3), "steps": steps, "paramset": kind,
           "h2d_bytes_per_step": 3 * 8 * n, "d2h_bytes_per_step": 2 * 8 * n + 8 * len(layout),
           "path": "optim.apply_update(host fp64 ParamSet): DMA w,g,m in (pinned in place), "
                   "fp64->fp32 on device, lars_step, fp32->fp64, DMA w,m back, dict(lambdas); "
                   "groups pipelined in parts (copy-back of part i overlaps copy-in of part i+1)"}
    if cpu_ms:
        out["speedup_vs_cpu_reference"] = round(cpu_ms / (med * 1e3), 2)
    return out


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import numpy as np
    from paper_1709_05011_b200 import layouts
    layout = layouts.get(args.workload)
    n_total = layouts.total_params(layout)
    if world > 1:
        # bounded sample: the reference DP step (all_reduce of P gradient
        # sets + /B + P x apply_update, cluster.py:146-153) on a prefix of
        # the groups holding ~1/P of the parameters
        sample, acc = [], 0
        for item in layout:
            sample.append(item)
            acc += int(np.prod(item[1]))
            if acc >= n_total / world:
                break
    else:
        sample = layout
    n = layouts.total_params(sample)
    rng = np.random.default_rng(1)
    grad_sets = [{name: rng.standard_normal(tuple(s)) for name, s, _ in sample}
                 for _ in range(world)] if world > 1 else None
    ref = stock_reference()
    if ref is not None:
        # the unmodified reference through its own public API: cluster.all_reduce,
        # `/ b`, ParamSet.set_grads + optim.apply_update per replica
        # (cluster.global_step, cluster.py:145-153, minus the model)
        hp = ref.optim.HyperParams(**_recipe_kw())
        replicas = [_stock_paramset(ref, sample, 0) for _ in range(world)]

        def step():
            if world > 1:
                summed = ref.cluster.all_reduce(grad_sets)
                mean = {k: v / GLOBAL_BATCH for k, v in summed.items()}
                for r in replicas:
                    r.set_grads(mean)
            for r in replicas:
                ref.optim.apply_update(r, hp, 0.1)
        kind, threads = "reference", 1
        impl_desc = "stock batchlab (baseline/_ref) through its public API"
    else:
        from oracle import lars_oracle as orc
        threads = os.cpu_count() or 1
        hp = _HP()
        replicas = [_oracle_groups(sample, 0) for _ in range(world)]
        ports = [orc.ThreadedPort(r, threads) for r in replicas]

        def step():
            if world > 1:
                summed = orc.all_reduce(grad_sets)
                mean = {k: v / GLOBAL_BATCH for k, v in summed.items()}
                for r in replicas:
                    for g in r:
                        np.copyto(g.grad, mean[g.name])
            for p in ports:
                p.apply_update(hp, 0.1)
        kind = "port"
        impl_desc = f"oracle port (ThreadedPort, {threads} threads)"

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    ms = sum(times) / len(times) * 1e3
    value = BYTES_PER_PARAM * n / (ms * 1e-3) / 1e9
    sample_desc = (f"{'reference DP step (all_reduce + /B + P x update) on ' if world > 1 else ''}"
                   f"{len(sample)} groups / {n} params of {args.workload}, fp64 numpy, "
                   f"{impl_desc}")
    line = {
        "impl": "reference",
        "metric": "LARS step HBM GB/s (algorithmic 20 B/param; % of roofline in 'roofline')",
        "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, layout, world),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads,
                         "kind": kind, "sample": sample_desc, "cpu_model": cpu_model(),
                         "host_threads": os.cpu_count()},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
