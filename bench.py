"""Benchmark: correlator time-to-solution of the BASELINE.json configs[1] workload.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {cc,reference}] [--config c2]
Under torchrun (N > 1) every rank runs one TIME part (Lt/N time slices, no replication)
and the per-slice correlator sums are all-reduced over NCCL (§8(e)); rank 0 prints ONE
JSON line.  See DESIGN.md §Measurement for every field.

One step = one pass of the hot path over the workload:
  value: cc_execute (plan replay: every contraction + TR + correlator sums; graph mode) with
         the leaves already resident in HBM, + the NCCL all-reduce when N > 1;
  e2e:   the public API from pinned host buffers: cc_load_dag + cc_schedule (tree scheduler
         + LRU plan) + cc_set_leaf + cc_execute (H2D of every leaf inside) + correlator D2H.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import dags, rng as srng  # noqa: E402

FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")


def workload(name):
    if name == "c2":
        return dags.config_c2()
    if name == "c1":
        return dags.config_c1()
    if name == "c3":
        return dags.config_c3()
    if name == "c4":   # diagnostic (the bench's c4 record builds its own): the two-baryon DAG
        return dags.config_c4()
    if name.startswith("c5:"):   # diagnostic: c5 at a given N, e.g. c5:N=256 (not a bench line)
        return dags.config_c5(**{k: int(v) for k, v in (x.split("=") for x in name[3:].split(","))})
    if name.startswith("c2:"):   # diagnostic variants of c2, e.g. c2:n_loop4=192 (not bench lines)
        return dags.config_c2(**{k: int(v) for k, v in (x.split("=") for x in name[3:].split(","))})
    if name == "c2t":   # diagnostic: c2's trace stage alone (not a bench line)
        return dags.config_traces()
    if name == "c2s":
        return dags.config_c2(N=64, Lt=16, n_loop4=100, n_loop2=8)
    raise SystemExit("unknown config " + name)


def leaf_sigma(w, op):
    return srng.meson_sigma(w.N) if op == dags.LEAF_M else srng.baryon_sigma(w.N, w.S)


def leaf_shape(w, op):
    return (w.Lt, w.N, w.N) if op == dags.LEAF_M else (w.Lt, w.S, w.N, w.N, w.N)


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clocks + throttle reasons sampled every 5 ms during the timed region (NVML; the
    nvidia-smi CLI as a fallback, 100 ms)."""
    # NVML clocks-event-reason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.sm = []
        self.mx = None
        self.reasons = set()
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.th = threading.Thread(target=self._poll, daemon=True)
            self.th.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                f = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = f(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.th.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = list(self.sm), self.mx, set(self.reasons)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml 5 ms" if self.nvml else "nvidia-smi 100 ms"}


# ---------------------------------------------------------------------------------------------
def oracle_baseline(w, max_seconds=20.0):
    """The oracle as it stands (oracle/values.py, numpy complex128) on this host's cores,
    over a bounded sample of time slices; returns (seconds for the whole workload, sample)."""
    from oracle import values
    from oracle.dag import Dag
    from threadpoolctl import threadpool_info
    dag = Dag(w)
    ops = {u: n.op for u, n in dag.nodes.items()}
    cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    done, t_spent, t = 0, 0.0, 0
    chunk = max(1, w.Lt // 16)
    while t < w.Lt and t_spent < max_seconds:
        t1 = min(w.Lt, t + chunk)
        leaves = {u: values.synthetic_leaf(w, u, ops[u], (t, t1)) for u in dag.nodes if not dag.nodes[u].child}
        t0 = time.perf_counter()
        roots = values.evaluate(dag, lambda u: leaves[u])
        values.correlators(dag, roots)
        t_spent += time.perf_counter() - t0
        done += t1 - t
        t = t1
    full = t_spent * w.Lt / done
    return full, cores, "%d of %d time slices, all %d trees (per-slice independence: x%.2f)" % (
        done, w.Lt, len(w.trees), w.Lt / done)


def run_reference(args, rank):
    w = workload(args.config)
    if rank != 0:
        return
    steps = []
    for i in range(args.warmup + args.steps):
        full, cores, sample = oracle_baseline(w, max_seconds=max(2.0, 60.0 / (args.warmup + args.steps)))
        if i >= args.warmup:
            steps.append(full)
    v = float(np.mean(steps))
    line = {"impl": "reference", "metric": "correlator time-to-solution", "value": v, "unit": "s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(w, args),
            "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: re-run this command as N ranks under
    torch.distributed.run on 127.0.0.1 (one process per GPU), NCCL communicator lines on
    (NCCL_DEBUG=INFO, INIT subsystem) unless the caller set them.  Returns the launcher's
    exit code; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def config_dict(w, args):
    return {"workload": "%s (BASELINE.json configs[1]: pi-pi I=2 correlator set, %d graphs sharing meson "
                        "nodes, N=%d, Lt=%d)" % (w.name, len(w.trees), w.N, w.Lt),
            "N": w.N, "Lt": w.Lt, "S": w.S, "trees": len(w.trees), "scheduler": "tree (Alg. 4-8)",
            "parallelism": "time-slice split x%d + %s all-reduce of correlators" % (
                args.gpus, getattr(args, "dist_backend", "nccl").upper()) if args.gpus > 1 else "single GPU",
            "l2": "flushed (256 MiB write) before every timed step; inputs (512 MiB of leaves) exceed L2",
            "leaves": "value: device-resident (HBM); e2e: pinned host, H2D inside the step"}


# ---------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cc", choices=["cc", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo to test N ranks on fewer GPUs")
    ap.add_argument("--c4", type=int, default=None,
                    help="1: add the c4 eviction-workload record (default: on at N=1, off at N>1); 0: off")
    ap.add_argument("--c4-steps", type=int, default=1, help="timed executes per c4 schedule")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    if args.c4 is None:
        args.c4 = 1 if world == 1 and args.config == "c2" else 0
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2511_02257_b200 import cc
    from paper_2511_02257_b200.dist import allreduce_correlators

    local_dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    w = workload(args.config)
    streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
    cs = streams[0]
    arena = torch.empty(6 << 30, dtype=torch.uint8, device=dev)
    ctx = cc.Context(local_dev, arena, streams=streams)
    ctx.load_workload(w)
    if world > 1:
        ctx.partition(world, rank, cc.PART_TIME)   # this rank's time slices [t0, t1)
    t0, t1 = ctx.part_time_range()
    Lt_p = t1 - t0

    # leaves: device-resident copy of this rank's slices (value) + pinned host full leaves (e2e)
    leaf_ops = [(n[0], n[1]) for n in w.nodes if n[1] in (dags.LEAF_M, dags.LEAF_B)]
    dev_leaves, host_leaves = {}, {}
    for (u, op) in leaf_ops:
        shape = leaf_shape(w, op)
        per_t = int(np.prod(shape[1:]))
        d = torch.empty(2 * Lt_p * per_t, dtype=torch.float64, device=dev)
        ctx.fill_synthetic(d, Lt_p * per_t, w.data_seed, u, t0 * per_t, w.leaf_mode, leaf_sigma(w, op))
        dev_leaves[u] = d
        h = torch.empty(2 * w.Lt * per_t, dtype=torch.float64, pin_memory=True)
        full = torch.empty(2 * w.Lt * per_t, dtype=torch.float64, device=dev)
        ctx.fill_synthetic(full, w.Lt * per_t, w.data_seed, u, 0, w.leaf_mode, leaf_sigma(w, op))
        torch.cuda.synchronize()
        h.copy_(full)
        del full
        host_leaves[u] = h
    torch.cuda.synchronize()

    # ---- value: plan replay with resident leaves --------------------------------------------------
    order, pst = ctx.schedule(cc.CC_TREE)
    for u, d in dev_leaves.items():
        ctx.set_leaf_device(u, d)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ptr, n_corr, corr_ids = None, None, None
    corr_full = None

    def step_value():
        ctx.execute_async(cc.EXEC_GRAPH)
        if world > 1:
            with torch.cuda.stream(cs):
                allreduce_correlators(corr_view, t0, t1, w.Lt, out=corr_full)

    # first execute builds the graph; bind the correlator buffer view for the all-reduce
    ctx.execute(cc.EXEC_GRAPH)
    ptr, n_corr, corr_ids = ctx.correlator_device_ptr()
    corr_view = _device_view(ptr, (n_corr, Lt_p), dev)
    corr_full = torch.zeros((n_corr, w.Lt), dtype=torch.complex128, device=dev)

    for _ in range(args.warmup):
        step_value()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(cs):
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            step_value()
            e1.record(cs)
            times.append((e0, e1))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_s = [a.elapsed_time(b) * 1e-3 for a, b in times]
    t_value = float(np.sum(step_s))

    # ---- roofline of the dominant kernel.  The step runs as ONE persistent launch of
    # df_worker (every MM1 tile and TR_MM block pair of the plan) + a tiny correlator kernel.
    # Launch duration: CUDA events on the compute stream around stream-mode replays (flags 0:
    # memset + df_worker + correlate; the worker is > 99 % of it), L2 flushed before each,
    # right after the timed region. ---------------------------------------------------------------
    ex0 = ctx.execute(0)
    n_kernels_step = ctx.execute(cc.EXEC_GRAPH)["n_kernels"]
    wt = []
    for _ in range(3):
        with torch.cuda.stream(cs):
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        ctx.execute_async(0)
        e1.record(cs)
        e1.synchronize()
        wt.append(e0.elapsed_time(e1) * 1e-3)
    worker_t = float(np.median(wt))
    step_flops = ex0["flops"]
    # FP64 work the pipes execute: GEMMs run as 3M (6 real flops per complex MAC, DESIGN V-3)
    gemm_fl = sum(8.0 * Lt_p * (w.N ** 3 if n[1] == dags.MM1 else w.S * w.N ** 4)
                  for n in w.nodes if n[1] in (dags.MM1, dags.BM1, dags.BB2))
    pipe_flops = step_flops - gemm_fl + 0.75 * gemm_fl
    step_hbm = ex0["hbm_bytes"]
    # component kernels alone (op-by-op path, flags 4/8: the plan's MM1 / TR_MM launches of the
    # stand-alone kernels replayed as CUDA graphs): kernel quality, not the step
    g_s = t_s = 0.0
    g_n = t_n = 0
    ctx.execute(cc.EXEC_ONLY_GEMM)
    ctx.execute(cc.EXEC_ONLY_TRACE)
    for _ in range(3):
        with torch.cuda.stream(cs):
            flush.zero_()
        eg = ctx.execute(cc.EXEC_ONLY_GEMM)
        g_s += eg["seconds"]
        g_n += eg["n_kernels"]
        with torch.cuda.stream(cs):
            flush.zero_()
        et = ctx.execute(cc.EXEC_ONLY_TRACE)
        t_s += et["seconds"]
        t_n += et["n_kernels"]
    mm1_avg = g_s / max(g_n, 1)
    tr_avg = t_s / max(t_n, 1)
    Lt_k, N = Lt_p, w.N
    mm1_flops = 8.0 * Lt_k * N ** 3
    step_mean = t_value / args.steps
    ozaki = ozaki_component(ctx, cs, flush, dev, [(Lt_k, N), (2, 1024)]) if rank == 0 else None

    # ---- e2e: the public API from pinned host buffers ------------------------------------------------
    arena2 = torch.empty(6 << 30, dtype=torch.uint8, device=dev)
    ctx2 = cc.Context(local_dev, arena2, streams=streams)
    e2e = []
    h2d_step = d2h_step = 0

    # time-to-solution: from cc_execute with the leaves in pinned host memory
    # to the correlators on the host.  Loading the DAG and scheduling happen before the timed
    # region (reported as sched_ms); re-scheduling invalidates the plan, so every timed
    # execute also prepares its physical plan, dataflow queues and tensor maps.
    sched_ms = []

    def prepare_e2e():
        t0 = time.perf_counter()
        ctx2.load_workload(w)
        if world > 1:
            ctx2.partition(world, rank, cc.PART_TIME)
        ctx2.schedule(cc.CC_TREE)
        sched_ms.append((time.perf_counter() - t0) * 1e3)
        for u, h in host_leaves.items():
            ctx2.set_leaf(u, h)

    corr_full2 = torch.zeros((n_corr, w.Lt), dtype=torch.complex128, device=dev)
    host_corr = torch.empty((n_corr, w.Lt), dtype=torch.complex128, pin_memory=True)

    def step_e2e():
        # solve (this rank's time slices), sum the ranks' correlators over NCCL, read to host
        st = ctx2.execute(0)
        if world == 1:
            ctx2.correlators(host_corr)        # one copy through the C ABI
            return st, host_corr
        ptr2, _, _ = ctx2.correlator_device_ptr()
        view2 = _device_view(ptr2, (n_corr, Lt_p), dev)
        with torch.cuda.stream(cs):
            full = allreduce_correlators(view2, t0, t1, w.Lt, out=corr_full2)
            host_corr.copy_(full, non_blocking=True)
        cs.synchronize()
        return st, host_corr

    for _ in range(max(1, args.warmup)):
        prepare_e2e()
        step_e2e()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    copy_ms = []
    for _ in range(args.steps):
        prepare_e2e()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        st, out = step_e2e()
        e1.record(cs)
        e1.synchronize()
        e2e.append(e0.elapsed_time(e1) * 1e-3)
        copy_ms.append(st["copy_seconds"] * 1e3)
        h2d_step = st["h2d_bytes"]
        d2h_step = st["d2h_bytes"] + n_corr * w.Lt * 16
    t_e2e = float(np.sum(e2e))
    del ctx2, arena2
    c4 = None
    if args.c4:
        if world == 1:
            try:
                c4 = c4_record(dev, local_dev, streams, args.c4_steps, world, rank)
            except Exception as e:      # the c2 line stands; the record says what failed
                c4 = {"error": "%s: %s" % (type(e).__name__, e)}
        else:                           # collectives inside: an exception on one rank must end the job
            c4 = c4_record(dev, local_dev, streams, args.c4_steps, world, rank)

    # max over ranks
    if world > 1:
        tt = torch.tensor([t_value, t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_value, t_e2e = float(tt[0]), float(tt[1])

    if rank == 0:
        peak, peak_src = fp64_peak()
        hbm_peak = measured_hbm()
        achieved = step_flops / worker_t / 1e12
        line = {
            "metric": "correlator time-to-solution", "value": t_value / args.steps, "unit": "s",
            "value_scope": "leaves already resident in HBM (contractions + traces + correlator sums); the "
                           "time to solution from pinned host leaves (H2D inside) is e2e",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_value / args.steps * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(w, args),
            "e2e": {"value": t_e2e / args.steps, "unit": "s", "h2d_bytes_per_step": int(h2d_step),
                    "d2h_bytes_per_step": int(d2h_step),
                    "how": "cc_execute (plan preparation + H2D of the pinned host leaves + dataflow worker) "
                           "+ correlators read back to the host, CUDA events on the compute stream; DAG load + "
                           "scheduling before the timed region",
                    "sched_ms": float(np.median(sched_ms)) if sched_ms else None,
                    "copies_done_ms": float(np.median(copy_ms)) if copy_ms else None,
                    "pcie_bound_s": (h2d_step + d2h_step) / 55.6e9},
            "gpu_launches": int(n_kernels_step * args.steps),
            "contraction_tflops": step_flops / step_mean / 1e12,
            "roofline": {"bound": "tensor",
                         "kernel": "df_worker (one persistent dataflow launch per step: every MM1 tile and "
                                   "TR_MM block pair of the plan; FP64 DMMA + DFMA)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "frac_note": "achieved counts the algorithmic 8 flops per complex MAC; the GEMMs execute the "
                                      "3M form (6), so frac can exceed 1 — the FP64 pipe's executed fraction is "
                                      "fp64_pipe.frac",
                         "traffic": ncu_traffic(), "peak_source": peak_src,
                         "algorithmic": {"flops_per_launch": step_flops, "hbm_bytes_per_launch": step_hbm},
                         "launch_ms": worker_t * 1e3,
                         "bound_ms": {"fp64": step_flops / (peak * 1e12) * 1e3,
                                      "hbm": step_hbm / (hbm_peak * 1e9) * 1e3},
                         "hbm_achieved_gbs": step_hbm / worker_t / 1e9,
                         "fp64_pipe": {"executed_tflops": pipe_flops / worker_t / 1e12,
                                       "frac": pipe_flops / worker_t / 1e12 / peak,
                                       "note": "achieved counts 8 flops per complex MAC (algorithmic); the "
                                               "GEMM k-tiles execute the 3M form (6), so the pipes run "
                                               "executed_tflops"},
                         "how": "CUDA events on the compute stream around stream-mode replays (df_worker + "
                                "memset + correlator kernel), L2 flushed before, 3 replays after the timed region; "
                                "achieved = algorithmic FP64 flops (8 per complex MAC) / launch time",
                         "components": {
                             "mm1_zgemm_alone": {"avg_us": mm1_avg * 1e6, "tflops": mm1_flops / mm1_avg / 1e12,
                                                 "frac": mm1_flops / mm1_avg / 1e12 / peak},
                             "tr_mm_alone": {"avg_us": tr_avg * 1e6,
                                             "gbs": 32.0 * Lt_k * N * N / tr_avg / 1e9,
                                             "frac": 32.0 * Lt_k * N * N / tr_avg / 1e9 / hbm_peak},
                             "mm1_ozaki_tcgen05": ozaki,
                             "how": "op-by-op path (cc_execute flags 4/8): the plan's MM1 / TR_MM launches of the "
                                    "stand-alone kernels replayed alone as CUDA graphs, L2 flushed before"}},
            "plan_by_scheduler": plan_by_scheduler(w),
            "plan": {"peak_bytes": pst["peak"], "transient_peak_bytes": pst["transient_peak"],
                     "evictions": pst["evictions"], "h2d_bytes": pst["h2d_bytes"], "d2h_bytes": pst["d2h_bytes"],
                     "sched_ms": pst["sched_seconds"] * 1e3, "plan_ms": pst["plan_seconds"] * 1e3},
            "clocks": clk.summary(),
        }
        if c4 is not None:
            line["c4_eviction_workload"] = c4
        if not args.no_cpu_baseline:
            full, cores, sample = oracle_baseline(w)
            line["cpu_baseline"] = {"value": full, "unit": "s", "cores": cores, "kind": "oracle", "sample": sample}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def plan_by_scheduler(w):
    """Host-only plans of the bench workload per scheduler (peak / transient peak; unbounded
    cap, so no evictions): the tree scheduler against the sibling and RS-GS-like ones."""
    from paper_2511_02257_b200 import cc
    out = {}
    c = cc.Context(-1)
    c.load_workload(w)
    for name in ("CC_TREE", "CC_SIBLING", "CC_RSGS"):
        st = c.schedule(getattr(cc, name))[1]
        out[name[3:].lower()] = {"peak_bytes": st["peak"], "transient_peak_bytes": st["transient_peak"],
                                 "sched_ms": st["sched_seconds"] * 1e3}
    c.close()
    return out


C4_RUNS = [   # (label, scheduler, next-use eviction)
    ("tree+next_use", "CC_TREE", True),
    ("tree+lru", "CC_TREE", False),
    ("sibling+lru", "CC_SIBLING", False),
    ("rsgs_like+lru", "CC_RSGS", False),
]


def c4_record(dev, local_dev, streams, steps, world=1, rank=0, pcie_gbs=55.6, pcie_d2h_gbs=57.2,
              lend_bytes=24 * 10 ** 9):
    """The paper's thesis workload (BASELINE configs[3]): the two-baryon DAG
    (2000 trees, N=128, S=64, Lt=1: 2 GiB baryon nodes) with the device pool capped at
    32e9 B so the plan evicts.  Each run: one warm-up (physical plan + pinned host pool built)
    and `steps` timed executions from host leaves to correlators on the host (the dataflow
    worker: FP64 DMMA GEMMs, copies overlapped through the flag protocol); the bytes the
    executor enqueued are compared with the oracle-parity plan's.
    N = 1: leaves in pinned host memory; tree scheduler with next-use and LRU eviction,
    sibling, and the RS-GS-like baseline.
    N > 1: each rank runs its TREES part (§8(e)) under its own 32e9 B cap with the peer-HBM
    tier of DESIGN E-10 (it evicts into the next rank's lent HBM, lend_bytes) and cross-GPU
    leaf sharing E-11 (each leaf crosses PCIe once per run, into its owner rank's HBM, inside
    the timed region; the other ranks copy it over NVLink); times are the max over ranks,
    bytes / evictions the sum.  Returns the record (rank 0)."""
    import torch
    from paper_2511_02257_b200 import cc
    w = dags.config_c4()
    cap = 32 * 10 ** 9
    # device memory this needs (arena + owned-leaf staging + lent tier), checked on every rank
    # before any collective so that no rank starts the record while another cannot
    need = (48 << 30) + ((34 << 30) // world + lend_bytes if world > 1 else 0)
    free = torch.tensor([float(torch.cuda.mem_get_info(dev)[0])], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(free, op=dist.ReduceOp.MIN)
    if float(free[0]) < need:
        return {"skipped": "needs %.1f GB of free device memory per rank, %.1f GB free" % (need / 1e9, float(free[0]) / 1e9)}
    arena = torch.empty(48 << 30, dtype=torch.uint8, device=dev)
    ctx = cc.Context(local_dev, arena, streams=streams)
    ctx.load_workload(w)
    owners = None
    if world > 1:
        ctx.partition(world, rank, cc.PART_TREES)
        owners = ctx.leaf_owners()
    t_setup = time.perf_counter()
    host, leaf_bytes = {}, {}
    tmp = None
    for n in w.nodes:
        if n[1] not in (dags.LEAF_M, dags.LEAF_B):
            continue
        cnt = int(np.prod(leaf_shape(w, n[1])))
        leaf_bytes[n[0]] = 16 * cnt
        if owners is not None and owners.get(n[0]) != rank:
            continue                               # another rank loads it (E-11)
        if tmp is None or tmp.numel() < 2 * cnt:
            tmp = torch.empty(2 * cnt, dtype=torch.float64, device=dev)
        d = tmp[:2 * cnt]
        ctx.fill_synthetic(d, cnt, w.data_seed, n[0], 0, w.leaf_mode, leaf_sigma(w, n[1]))
        h = torch.empty(2 * cnt, dtype=torch.float64, pin_memory=True)
        torch.cuda.synchronize()
        h.copy_(d)
        host[n[0]] = h
    del tmp
    torch.cuda.synchronize()
    shared, lent = None, None
    if world > 1:
        from paper_2511_02257_b200.dist import SharedLeaves, setup_peer_tier
        shared = SharedLeaves(ctx, leaf_bytes, host, dev)
        lent, tier_ptrs = setup_peer_tier(ctx, lend_bytes, dev)
    t_setup = time.perf_counter() - t_setup
    n_corr = len({t[0] for t in w.terms})
    host_corr = torch.empty((n_corr, w.Lt), dtype=torch.complex128, pin_memory=True)
    runs = {}
    # the DMMA dataflow worker (1.58 s on c4 at 48 GiB of arena; the Ozaki engine's leaf-form
    # cache needs headroom beyond the cap: 1.42-1.55 s at 60-100 GiB, 1.79 s at 48 GiB)
    flags = 0
    plan_runs = C4_RUNS if world == 1 else [("tree+next_use+peer_hbm", "CC_TREE", True)]
    for k, (label, algo, nu) in enumerate(plan_runs):
        t0 = time.perf_counter()
        if world == 1:
            _, st = ctx.schedule(getattr(cc, algo), cap_bytes=cap, evict_next_use=nu)
            for u, h in host.items():
                ctx.set_leaf(u, h)
        else:
            _, st = ctx.schedule(getattr(cc, algo), cap_bytes=cap, evict_next_use=nu, peer_cap_bytes=lend_bytes,
                                 peer_leaves=shared.ids)
        sched_s = time.perf_counter() - t0
        part = ctx.part_info()          # replicated share of a TREES part (reading M-3)
        # the schedule's own peak without a cap (what the paper's 2.1x compares): host only
        hctx = cc.Context(-1)
        hctx.load_workload(w)
        if world > 1:
            hctx.partition(world, rank, cc.PART_TREES)
        uncapped = hctx.schedule(getattr(cc, algo))[1]
        hctx.close()
        # warm-up of this plan: builds the physical plan and allocates its pinned host pool for
        # evicted intermediates (64 GB for the RS-GS-like plan), which a replay reuses
        if shared is not None:
            shared.stage()
        ctx.execute(flags)
        ts, ex, staged = [], None, 0
        for _ in range(steps):
            torch.cuda.synchronize()
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(streams[0])
            if shared is not None:
                staged = shared.stage()            # the owners' H2D of the shared leaves
            ex = ctx.execute(flags)
            ctx.correlators(host_corr)
            e1.record(streams[0])
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t = float(np.median(ts))
        st = dict(st)
        ex = dict(ex)
        st["h2d_bytes"] += staged                  # leaf staging is PCIe traffic of the run
        ex["h2d_bytes"] += staged
        if world > 1:
            import torch.distributed as dist
            keys = ("evictions", "h2d_bytes", "d2h_bytes", "p2p_in_bytes", "p2p_out_bytes")
            pv = torch.tensor([part["work"], part["replicated_work"], part["leaf_bytes"], part["replicated_leaf_bytes"]],
                              dtype=torch.float64, device=dev)
            dist.all_reduce(pv, op=dist.ReduceOp.SUM)
            part = dict(work=int(pv[0]), replicated_work=int(pv[1]), leaf_bytes=int(pv[2]),
                        replicated_leaf_bytes=int(pv[3]))
            v = torch.tensor([t] + [st[k] for k in keys] + [ex["h2d_bytes"], ex["d2h_bytes"], ex["p2p_in_bytes"],
                                                           ex["p2p_out_bytes"]], dtype=torch.float64, device=dev)
            tmax = v[:1].clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            dist.all_reduce(v, op=dist.ReduceOp.SUM)
            t = float(tmax[0])
            st.update({k: int(v[1 + i]) for i, k in enumerate(keys)})
            ex.update(h2d_bytes=int(v[6]), d2h_bytes=int(v[7]), p2p_in_bytes=int(v[8]), p2p_out_bytes=int(v[9]))
        # H2D and D2H use the two directions of the link (one link per GPU): the bound is the
        # busier direction
        pcie_bound = max(st["h2d_bytes"] / (pcie_gbs * 1e9), st["d2h_bytes"] / (pcie_d2h_gbs * 1e9)) / world
        runs[label] = {
            "e2e_s": t, "steps": steps, "sched_s": sched_s,
            "peak_bytes": st["peak"], "transient_peak_bytes": st["transient_peak"], "evictions": st["evictions"],
            "uncapped_peak_bytes": uncapped["peak"], "uncapped_transient_peak_bytes": uncapped["transient_peak"],
            "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"], "host_peak_bytes": st["host_peak_bytes"],
            "p2p_in_bytes": st.get("p2p_in_bytes", 0), "p2p_out_bytes": st.get("p2p_out_bytes", 0),
            "runtime_h2d_bytes": int(ex["h2d_bytes"]), "runtime_d2h_bytes": int(ex["d2h_bytes"]),
            "bytes_match_plan": int(ex["h2d_bytes"]) == st["h2d_bytes"] and int(ex["d2h_bytes"]) == st["d2h_bytes"]
            and int(ex.get("p2p_in_bytes", 0)) == st.get("p2p_in_bytes", 0),
            "pcie_bound_s": pcie_bound, "pcie_frac": pcie_bound / t,
            "fp64_flops": ex["flops"], "copies_done_s": ex["copy_seconds"],
            "replication": {"work_flops_over_8": part["work"], "replicated_work": part["replicated_work"],
                            "replicated_work_share": part["replicated_work"] / max(part["work"], 1),
                            "leaf_bytes": part["leaf_bytes"], "replicated_leaf_bytes": part["replicated_leaf_bytes"],
                            "note": "summed over ranks; reading M-3 (owner = part of the first selected tree)"}}
    ratios = {}
    if "rsgs_like+lru" in runs:
        base = runs["rsgs_like+lru"]
        for label in ("tree+next_use", "tree+lru", "sibling+lru"):
            r = runs[label]
            ratios[label] = {"time": base["e2e_s"] / r["e2e_s"],
                             "evictions": base["evictions"] / max(r["evictions"], 1),
                             "peak": base["peak_bytes"] / r["peak_bytes"],
                             "uncapped_peak": base["uncapped_peak_bytes"] / r["uncapped_peak_bytes"],
                             "bytes_moved": (base["h2d_bytes"] + base["d2h_bytes"]) / (r["h2d_bytes"] + r["d2h_bytes"])}
    if world > 1:
        dist.barrier()                              # every rank's executes are done
        shared.close()
        from paper_2511_02257_b200.dist import close_buffers
        close_buffers(tier_ptrs)
    leaf_bytes_total = sum(leaf_bytes.values())
    del ctx, arena, host, lent
    torch.cuda.empty_cache()
    return {"workload": "%s (BASELINE.json configs[3]: two-baryon system, %d graphs, N=%d, S=%d, Lt=%d; "
                        "device pool capped at 32e9 B)" % (w.name, len(w.trees), w.N, w.S, w.Lt),
            "cap_bytes": cap, "ranks": world,
            "split": "TREES parts, one per rank; peer-HBM tier (E-10, %d B lent per rank) + shared leaves (E-11)"
                     % lend_bytes if world > 1 else "none",
            "engine": "dataflow worker (FP64 DMMA 3M GEMMs; copies on their streams, flag-synchronised)",
            "leaves": "pinned host (%.1f GiB), H2D inside every timed execution" % (leaf_bytes_total / 2 ** 30),
            "pcie_gbs_measured": {"h2d": pcie_gbs, "d2h": pcie_d2h_gbs,
                                  "source": "profiles/r01_microbench_fp64_pcie.txt (pinned cudaMemcpyAsync)"},
            "setup_s": t_setup, "runs": runs, "rsgs_over_ours": ratios,
            "paper_context": "paper (Frontier/Summit-era GPUs, Redstar): up to 1.9x faster, 2.1x lower peak memory, "
                             "4.2x fewer evictions than RS-GS (P:31, P:944, P:979-982)"}


def _device_view(ptr, shape, dev):
    """A torch complex128 view of a device buffer owned by libcc (no copy)."""
    import torch
    n = int(np.prod(shape))

    class _Holder:
        __cuda_array_interface__ = {"shape": (n * 2,), "typestr": "<f8", "data": (ptr, False), "version": 2}
    t = torch.as_tensor(_Holder(), device=dev)
    return t.view(torch.complex128).view(*shape)


def int8_peak():
    """Dense INT8 tensor peak: measured bf16 (MEASURED_PEAKS.json, burst) x the guide's nominal
    INT8/BF16 ratio of 2 (4.5 / 2.25 PFLOP/s)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return 2.0 * float(json.load(f)["bf16_tflops"]), "2 x measured bf16 (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 4500.0, "nominal dense INT8 (B200_PROFILING.md)"


def ozaki_component(ctx, cs, flush, dev, shapes, slices=5):
    """MM1 on the tcgen05 INT8 Ozaki engine (cc_mm1_ozaki) at the given (Lt, N):
    split + GEMM time from CUDA events on the compute stream (L2 flushed before each launch,
    median of 5), FP64-equivalent TFLOP/s (8 per complex MAC) and INT8 tensor TOPS executed
    (slices(slices+1)/2 pair products of the 4M real embedding, 2 x 4 N^3 ops per slice)."""
    import torch
    from paper_2511_02257_b200 import cc
    out = []
    pk, src = int8_peak()
    for (Lt, N) in shapes:
        A = torch.empty(Lt * N * N * 2, dtype=torch.float64, device=dev)
        B = torch.empty_like(A)
        C = torch.empty_like(A)
        ctx.fill_synthetic(A, Lt * N * N, 11, 1, 0, 0, 1.0 / N)
        ctx.fill_synthetic(B, Lt * N * N, 11, 2, 0, 0, 1.0 / N)
        ws = torch.empty(cc.cc_mm1_ozaki_workspace_bytes(Lt, N, slices), dtype=torch.uint8, device=dev)
        ts = []
        for _ in range(7):
            with torch.cuda.stream(cs):
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            ctx.mm1_ozaki(A, B, C, Lt, N, slices, ws)
            e1.record(cs)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t = float(np.median(ts[2:]))
        int8_ops = 2.0 * (slices * (slices + 1) // 2) * 4.0 * Lt * N ** 3
        out.append({"Lt": Lt, "N": N, "slices": slices, "avg_us": t * 1e6,
                    "tflops_fp64_equiv": 8.0 * Lt * N ** 3 / t / 1e12, "int8_tops": int8_ops / t / 1e12,
                    "int8_frac": int8_ops / t / 1e12 / pk})
        del A, B, C, ws
    return {"runs": out, "int8_peak_tops": pk, "peak_source": src,
            "note": "not on the bench step (c2 runs MM1 on FP64 DMMA in df_worker); split kernels included"}


def fp64_peak():
    try:
        with open(FP64_PEAK_FILE) as f:
            d = json.load(f)
        return d["tflops"], d["source"]
    except (OSError, KeyError, ValueError):
        return 37.0, "fallback: DMMA microbenchmark of round 1 (profiles/r01_microbench_fp64_pcie.txt)"


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0   # B200_PROFILING.md fallback


def ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f).get("df_worker_traffic_bytes_per_launch")
    except (OSError, ValueError):
        return None


if __name__ == "__main__":
    main()
