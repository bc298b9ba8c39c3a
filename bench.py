#!/usr/bin/env python
"""Benchmark: P1 stiffness+load assembly (+ Dirichlet system) on B200.

One "step" = one pass of the hot path over the configuration's mesh, exactly
what solve_poisson builds before its solve (solver.hpp:226-242):
partition_boundary + assemble_blockwise + assemble_load + apply_neumann +
apply_dirichlet + submatrix(A, free, free) + b_f, INCLUDING the topology plan
(node -> element incidence lists) rebuilt from the raw arrays every step
(FL_REPLAN: a cold mesh, nothing cached across steps except device buffers).

  value      elements/s with inputs resident in HBM (CUDA events per step, max
             over ranks);
  e2e        the same through the C-ABI with HOST buffers: H2D of the mesh arrays
             from pinned memory, assembly, D2H of every output array;
  roofline   the dominant kernel (k_columns) against the measured HBM copy peak;
  cpu_baseline / --impl reference
             the reference's own CPU path (oracle/_ref = femlite compiled from
             its headers) on a bounded sample of the same workload family.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5]
       python bench.py --impl reference ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DEFAULT_CONFIG = "C5"
METRIC = "P1 stiffness+load assembly elements/sec and achieved HBM GB/s vs peak, 1/2/4/8 GPU"
UNIT = "elements/s"
L2_BYTES = 126 * 2 ** 20

# bounded CPU samples (same family, smaller n): ~10-30 s of reference work
CPU_SAMPLE_N = {"C1": 128, "C2": 512, "C3": 1024, "C4": 64, "C5": 64}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled
    every ~2 ms from a thread (the timed region can be a few ms), with
    nvidia-smi -lms 100 as the fallback when NVML is unavailable."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, reasons_mask)
        self._stop = threading.Event()
        self._thread = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            # CUDA_VISIBLE_DEVICES remaps ordinals: match the torch device by UUID
            import torch
            h = None
            uuid = getattr(torch.cuda.get_device_properties(self.device), "uuid", None)
            if uuid is not None:
                want = "GPU-" + str(uuid)
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(hi)
                    if (u.decode() if isinstance(u, bytes) else u) == want:
                        h = hi
                        break
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self._nv, self._h = pynvml, h
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._thread = threading.Thread(target=self._poll, daemon=True)
            self._thread.start()
        except Exception as e:  # pragma: no cover - box without NVML
            log(f"[bench] NVML unavailable ({e}); clocks unsampled")

    def _poll(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, self._max, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        self._stop.set()
        if self._thread:
            self._thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({n for _, _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "NVML, 2 ms polling in the timed region"}


# ---------------------------------------------------------------------------
# reference CPU path on a bounded sample
# ---------------------------------------------------------------------------
def cpu_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_reference(config: str, seconds_budget: float = 25.0, reps: int | None = None,
                  threads: int | None = None):
    """Time femlite's own solve_poisson pre-solve path (oracle/_ref) on a sample,
    on every host thread: the reference is single-threaded by construction, so T
    threads each run the whole path on the sample concurrently and the value is
    T x NT elements per wall-clock round (throughput with all host cores)."""
    from oracle import pyoracle as po
    from paper_1804_05156_b200 import configs
    if not po.have_ref():
        return None
    n = CPU_SAMPLE_N[config]
    cfg = configs.build(config, n=n)  # numpy-only generators: no libfemlite_b200.so here
    m = cfg.mesh
    coef = po.coefficient_c5(m.dim, m.nodes, m.elems) if cfg.coef else None
    f_kind = po.FIELD_SINSIN if cfg.f == "sinsin" else po.FIELD_CONST
    f_val = 0.0 if cfg.f == "sinsin" else float(cfg.f)
    T = threads or cpu_threads()
    secs = po.ref_time_system_mt(m.dim, m.nodes, m.elems, m.bd_flags, f_kind, f_val, coef, reps=1,
                                 threads=T)
    one = float(secs[0])
    if reps is None:
        reps = max(1, min(5, int(seconds_budget / max(one, 1e-6))))
    secs = po.ref_time_system_mt(m.dim, m.nodes, m.elems, m.bd_flags, f_kind, f_val, coef, reps=reps,
                                 threads=T)
    _, nnz, _ = po.ref_time_system(m.dim, m.nodes, m.elems, m.bd_flags, f_kind, f_val, coef, reps=1)
    med = float(np.median(secs))
    return {"value": T * m.num_elems() / med, "unit": UNIT, "cores": T, "kind": "reference",
            "seconds_per_step": med, "reps": int(len(secs)), "n_elems": T * m.num_elems(),
            "sample": (f"{cfg.description} (n={n}, NT={m.num_elems()}, nnz={nnz}) on each of {T} host "
                       "threads concurrently: femlite partition_boundary+assemble_blockwise+"
                       "assemble_load+apply_neumann+apply_dirichlet+submatrix+b_f (the reference is "
                       "single-threaded; T independent runs = throughput on all cores)")}


def workload_name(config: str) -> str:
    from paper_1804_05156_b200.configs import FULL_N
    desc = {"C1": "unit_square:{n}", "C2": "lshape:{n} jittered", "C3": "unit_square:{n} permuted",
            "C4": "unit_cube:{n}", "C5": "unit_cube:{n} permuted+coef"}[config]
    return f"{config}: " + desc.format(n=FULL_N[config])


def run_reference_impl(args, rank: int, world: int):
    if rank != 0:
        return
    from oracle import pyoracle as po
    if not po.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    # one round = the sample assembled on every host thread at once; W + K rounds
    base = cpu_reference(args.config, reps=1)
    from paper_1804_05156_b200 import configs
    cfg = configs.build(args.config, n=CPU_SAMPLE_N[args.config])
    m = cfg.mesh
    coef = po.coefficient_c5(m.dim, m.nodes, m.elems) if cfg.coef else None
    f_kind = po.FIELD_SINSIN if cfg.f == "sinsin" else po.FIELD_CONST
    f_val = 0.0 if cfg.f == "sinsin" else float(cfg.f)
    secs = po.ref_time_system_mt(m.dim, m.nodes, m.elems, m.bd_flags, f_kind, f_val, coef,
                                 reps=args.warmup + args.steps, threads=base["cores"])
    per_step = list(secs[args.warmup:])
    ms = 1e3 * float(np.mean(per_step))
    value = base["n_elems"] / (ms * 1e-3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            # the same workload as our arm's line; each step times a bounded sample of
            # it (the rate in elements/s is per element: see cpu_baseline.sample and
            # profiles/ for the full-size single-thread check)
            "config": {"workload": workload_name(args.config), "sample": base["sample"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": base["cores"], "kind": "reference",
                             "sample": base["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# GPU path
# ---------------------------------------------------------------------------
def load_traffic(config: str):
    """ncu dram bytes (read + write) per launch of the numeric phase, from profiles/."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        return json.load(fh).get(config)


def run_ours(args, rank: int, world: int):
    import ctypes as C

    import torch
    import torch.distributed as dist

    os.environ.setdefault("FL_PROFILE", "1")
    import paper_1804_05156_b200 as fl
    from paper_1804_05156_b200 import _lib, configs
    from paper_1804_05156_b200.mesh import DeviceMesh
    from paper_1804_05156_b200.shard import column_ranges

    # one process per GPU; FL_BENCH_BACKEND=gloo is a functional check of the
    # sharded path on fewer GPUs (ranks share a device; its numbers mean nothing)
    dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    L = _lib.lib()
    ctx = fl.Context(dev)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream.cuda_stream)

    t0 = time.time()
    cfg = configs.build(args.config, f_mode="samples")
    m = cfg.mesh
    N, NT, d = m.num_nodes(), m.num_elems(), m.dim
    c0, c1 = column_ranges(N, world)[rank]
    log(f"[bench] rank {rank}/{world} {args.config}: {cfg.description} N={N} NT={NT} "
        f"columns [{c0}, {c1}) built in {time.time() - t0:.1f}s")

    # device-resident inputs (uploaded once, untimed); this rank's column range
    dm = DeviceMesh(ctx, m)
    if world > 1:
        dm.set_columns(c0, c1)
    res = fl.AssemblyResult(ctx)
    what = _lib.OUT_SYSTEM | _lib.REPLAN

    ff, k1 = fl.api._field_struct(cfg.f, m, "load")
    fc, k2 = fl.api._field_struct(cfg.coef, m, "coef")
    fd, k3 = fl.api._field_struct(cfg.g_dirichlet, m, "dirichlet")
    fn, k4 = fl.api._field_struct(cfg.g_neumann, m, "neumann")
    f_dev = None
    if ff.kind == _lib.FIELD_SAMPLES:  # stage samples on the device once
        f_dev = torch.from_numpy(np.asarray(k1)).to(f"cuda:{dev}")
        ff.mem, ff.samples = _lib.MEM_DEVICE, f_dev.data_ptr()

    counts = torch.zeros(4, dtype=torch.int64, device=f"cuda:{dev}")
    all_counts = [torch.zeros(4, dtype=torch.int64, device=f"cuda:{dev}") for _ in range(world)]

    def step():
        _lib.check(L.fl_assemble(ctx.handle, dm.handle, C.byref(ff), C.byref(fc), C.byref(fd),
                                 C.byref(fn), what, res.handle), "fl_assemble")
        if world > 1:  # the nnz-offset exchange (NCCL all_gather on the same stream)
            _lib.check(L.fl_result_counts_async(res.handle, counts.data_ptr()))
            dist.all_gather(all_counts, counts)
            torch.cumsum(torch.stack(all_counts), dim=0)

    flush = None
    ws_bytes = configs.system_bytes(d, N, NT, 0, 0, 0)
    if ws_bytes < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=f"cuda:{dev}")

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
            sz = res.sizes()
        ctx.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = ctx.launch_count()
        clocks = ClockSampler(dev)
        clocks.start()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        phase, kph = [], []
        for k in range(args.steps):
            if flush is not None:
                flush.fill_(k)
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            sz = res.sizes()  # synchronises; resolves the phase events
            phase.append(ctx.last_timings())
            kph.append(ctx.last_kernel_timings())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks.stop()
        launches = ctx.launch_count() - launches0
        # the same step on the mesh's cached plan (repeated assemblies on one mesh:
        # time stepping, Newton, coefficient updates) -- reported beside the
        # headline, which rebuilds the plan every step like the reference
        cached = []
        if world == 1 and not args.no_cached:
            for _ in range(args.warmup):
                _lib.check(L.fl_assemble(ctx.handle, dm.handle, C.byref(ff), C.byref(fc), C.byref(fd),
                                         C.byref(fn), _lib.OUT_SYSTEM, res.handle), "fl_assemble")
                res.sizes()
            for k in range(args.steps):
                if flush is not None:
                    flush.fill_(k)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _lib.check(L.fl_assemble(ctx.handle, dm.handle, C.byref(ff), C.byref(fc), C.byref(fd),
                                         C.byref(fn), _lib.OUT_SYSTEM, res.handle), "fl_assemble")
                e1.record(stream)
                res.sizes()
                cached.append((e0, e1))
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms_local = float(np.mean(step_ms))
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        gathered = torch.stack(all_counts).cpu().numpy()
    col_ms = float(np.mean([p[2] for p in phase]))
    plan_ms = float(np.mean([p[0] for p in phase]))
    mark_ms = float(np.mean([p[1] for p in phase]))
    rec_ms, kern_ms, place_ms = (float(np.mean([p[i] for p in kph])) for i in range(3))

    # sizes: this rank's shard; global totals from the exchange
    nnz_l, nnz_ff_l, n_free = int(sz.nnz), int(sz.nnz_ff), int(sz.n_free)
    ncol_l, nfree_l = int(sz.n), int(sz.n_free_cols)
    nnz, nnz_ff = (int(gathered[:, 2].sum()), int(gathered[:, 3].sum())) if world > 1 else (nnz_l, nnz_ff_l)
    b_sl = configs.algorithmic_bytes(d, N, NT, nnz)
    b_sys = configs.system_bytes(d, N, NT, nnz, n_free, nnz_ff)
    f_bytes = 8 * NT * (d + 1) if ff.kind == _lib.FIELD_SAMPLES else 0
    # the column kernel's own compulsory bytes (this rank): label-plan keys and
    # relabelled elements read once (the share of the elements touching the
    # rank's columns), label-ordered node records of every node and the per-label
    # counts read once, 16-byte staged entries and per-node vector records written once
    frac_el = 1.0 if world == 1 else min(1.0, 1.0 - (1.0 - ncol_l / max(N, 1)) ** (d + 1))
    kern_bytes = (int(frac_el * 4 * (d + 1) * NT) + 4 * (d + 1) * int(NT * ncol_l / max(N, 1)) + f_bytes
                  + 32 * N + 4 * ncol_l + 16 * nnz_l + 32 * ncol_l)
    peak, peak_kind = peaks()
    # achieved = B_SL / t, t = the measured assembly (the whole step)
    achieved = b_sl / (ms * 1e-3) / 1e9
    traffic = load_traffic(args.config) if world == 1 else None

    # ---- optional verification gather to rank 0 (untimed): grouped NCCL
    # send/recv of every shard into the global CSC (gloo: CPU tensors) ----
    if args.dump_gather and world > 1:
        from paper_1804_05156_b200.shard import ShardInfo, exclusive_offsets, gather_csc_to_root
        info = ShardInfo(rank, world, c0, c1, gathered, exclusive_offsets(gathered))
        tdev = f"cuda:{dev}" if os.environ.get("FL_BENCH_BACKEND", "nccl") == "nccl" else "cpu"
        loc = []
        for which, dt, cnt in ((_lib.A_COL_PTR, torch.int32, ncol_l + 1), (_lib.A_ROW_IDX, torch.int32, nnz_l),
                               (_lib.A_VALUES, torch.float64, nnz_l)):
            t = torch.empty(max(cnt, 1), dtype=dt, device=f"cuda:{dev}")
            _lib.check(L.fl_result_copy(res.handle, which, t.data_ptr(), t.numel() * t.element_size(),
                                        _lib.MEM_DEVICE))
            loc.append(t[:cnt])
        ctx.synchronize()  # the copies ran on the library's stream
        loc = [t.to(tdev) for t in loc]
        torch.cuda.synchronize()
        out = gather_csc_to_root(info, *loc)
        if rank == 0:
            cp, ri, va = (x.cpu().numpy() for x in out)
            np.savez(args.dump_gather, col_ptr=cp, row_idx=ri, values=va, config=args.config)
            log(f"[bench] gathered the {world}-shard CSC on rank 0 -> {args.dump_gather}")

    # ---- e2e through the C-ABI with host buffers (pinned) ----
    e2e = None
    if not args.no_e2e:
        del res, dm  # release the device-resident run's buffers before the pipeline
        ctx.synchronize()
        e2e = run_e2e(args, cfg, torch, fl, _lib, L, C, dev, (c0, c1) if world > 1 else None)
        if world > 1:
            t = torch.tensor([e2e["ms_per_step"]], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["ms_per_step"] = float(t.item())
            e2e["value"] = NT / (e2e["ms_per_step"] * 1e-3)

    line = None
    if rank == 0:
        value = NT / (ms * 1e-3)  # the whole mesh, assembled by all ranks together
        cpu = None if args.no_cpu_baseline else cpu_reference(args.config)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator meshes, SURVEY.md §8(d) recipes)",
            "config": {"workload": workload_name(args.config), "n_nodes": N,
                       "n_elems": NT, "nnz": nnz, "nnz_ff": nnz_ff, "n_free": n_free,
                       "step": "plan+partition+stiffness+load+dirichlet+A_ff+b_f",
                       "l2": ("flushed between steps (256 MB write)" if flush is not None
                              else "inputs larger than L2"),
                       "parallelism": (f"row-sharded x{world} (contiguous column ranges; NCCL "
                                       "all_gather of nnz counts)" if world > 1 else "1 GPU"),
                       "f": str(cfg.f) if not isinstance(cfg.f, np.ndarray) else "host samples",
                       "coef": str(cfg.coef)},
            "hbm_gbs_step": b_sys / (ms * 1e-3) / 1e9,
            "bytes": {"B_SL": b_sl, "B_sys": b_sys, "f_samples": f_bytes, "column_kernel": kern_bytes},
            "phases_ms": {"plan": plan_ms, "partition": mark_ms, "numeric": col_ms,
                          "element_records": rec_ms, "column_kernel": kern_ms, "placement": place_ms},
            "roofline": {"bound": "hbm",
                         "kernel": "the whole step (fl_assemble), SURVEY.md §8(d): achieved = B_SL / ms_per_step",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "algorithmic_bytes": b_sl,
                         "traffic": traffic.get("step_dram_bytes") if traffic else None,
                         "traffic_source": traffic.get("source") if traffic else None,
                         "b_sys_frac": b_sys / (ms * 1e-3) / 1e9 / peak,
                         "dominant_kernel": {
                             "name": "k_columns4 (label-space column kernel)",
                             "ms": kern_ms, "share_of_step": kern_ms / ms if ms > 0 else None,
                             "compulsory_bytes": kern_bytes,
                             "achieved": kern_bytes / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else None,
                             "frac": kern_bytes / (kern_ms * 1e-3) / 1e9 / peak if kern_ms > 0 else None,
                             "traffic": traffic.get("kernel_dram_bytes") if traffic else None}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_single": e2e["single_call"] if e2e else None,
            "cached_plan": ({"value": NT / (float(np.mean([a.elapsed_time(b) for a, b in cached])) * 1e-3),
                             "unit": UNIT, "ms_per_step": float(np.mean([a.elapsed_time(b) for a, b in cached])),
                             "step": "partition+stiffness+load+dirichlet+A_ff+b_f on the cached plan"}
                            if cached else None),
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        if args.traffic:
            line["roofline"]["traffic"] = float(args.traffic)
        if line["roofline"]["traffic"]:
            # the DRAM bytes the step's kernels actually move (ncu) over the step time
            tg = line["roofline"]["traffic"] / (ms * 1e-3) / 1e9
            line["roofline"]["traffic_gbs"] = tg
            line["roofline"]["traffic_frac"] = tg / peak
        print(json.dumps(line))
    return line


def run_e2e(args, cfg, torch, fl, _lib, L, C, dev, cols=None):
    """End to end through the C-ABI from pinned host memory, per step: upload the
    mesh arrays (+ samples), assemble, synchronise for the sizes, copy every
    output array back.  `--e2e-depth` fl_ctx objects (each with its own stream,
    mesh and result) run consecutive steps as a pipeline -- step k's outputs
    stream back while step k+1 uploads/computes -- the way a caller processing a
    stream of meshes would use the API.  Throughput = steps / wall time."""
    m = cfg.mesh
    N, NT, d = m.num_nodes(), m.num_elems(), m.dim
    depth = max(1, args.e2e_depth)

    def pinned(a):
        t = torch.empty(a.shape, dtype={np.float64: torch.float64, np.int32: torch.int32,
                                        np.int8: torch.int8}[a.dtype.type], pin_memory=True)
        t.numpy()[...] = a
        return t

    h_nodes, h_elems, h_flags = pinned(m.nodes), pinned(m.elems), pinned(m.bd_flags)
    f_arr = np.asarray(cfg.f) if isinstance(cfg.f, np.ndarray) else None
    h_f = pinned(f_arr) if f_arr is not None else None
    ff, _k1 = fl.api._field_struct(cfg.f if f_arr is None else None, m, "load")
    if f_arr is not None:
        ff.kind, ff.mem, ff.samples, ff.n_samples = _lib.FIELD_SAMPLES, _lib.MEM_HOST, h_f.data_ptr(), f_arr.size
    fc, _k2 = fl.api._field_struct(cfg.coef, m, "coef")
    fd, _k3 = fl.api._field_struct(cfg.g_dirichlet, m, "dirichlet")
    fn, _k4 = fl.api._field_struct(cfg.g_neumann, m, "neumann")

    slots = []
    for _ in range(depth):
        ctx = fl.Context(dev)
        hmesh = C.c_void_p()
        _lib.check(L.fl_mesh_create(ctx.handle, d, N, NT, h_nodes.data_ptr(), h_elems.data_ptr(),
                                    h_flags.data_ptr(), _lib.MEM_HOST, C.byref(hmesh)))
        if cols is not None:
            _lib.check(L.fl_mesh_set_columns(ctx.handle, hmesh, cols[0], cols[1]))
        slots.append({"ctx": ctx, "mesh": hmesh, "res": fl.AssemblyResult(ctx), "outs": None})

    def issue(sl):
        ctx, hmesh = sl["ctx"], sl["mesh"]
        _lib.check(L.fl_mesh_set_nodes(ctx.handle, hmesh, h_nodes.data_ptr(), _lib.MEM_HOST))
        _lib.check(L.fl_mesh_set_elems(ctx.handle, hmesh, h_elems.data_ptr(), _lib.MEM_HOST))
        _lib.check(L.fl_mesh_set_flags(ctx.handle, hmesh, h_flags.data_ptr(), _lib.MEM_HOST))
        _lib.check(L.fl_assemble(ctx.handle, hmesh, C.byref(ff), C.byref(fc), C.byref(fd),
                                 C.byref(fn), _lib.OUT_SYSTEM | _lib.REPLAN, sl["res"].handle))

    def drain(sl):
        res = sl["res"]
        sz = res.sizes()
        if sl["outs"] is None:
            n, nf = sz.n, sz.n_free_cols  # this rank's columns (all of them at N=1)
            spec = [(_lib.A_COL_PTR, torch.int32, n + 1), (_lib.A_ROW_IDX, torch.int32, sz.nnz),
                    (_lib.A_VALUES, torch.float64, sz.nnz), (_lib.B, torch.float64, n),
                    (_lib.U0, torch.float64, n), (_lib.B_MOD, torch.float64, n),
                    (_lib.DIR_NODES, torch.int32, sz.n_dir), (_lib.FREE_NODES, torch.int32, sz.n_free),
                    (_lib.AFF_COL_PTR, torch.int32, nf + 1),
                    (_lib.AFF_ROW_IDX, torch.int32, sz.nnz_ff),
                    (_lib.AFF_VALUES, torch.float64, sz.nnz_ff), (_lib.B_F, torch.float64, nf)]
            sl["outs"] = [(w, torch.empty(max(c, 1), dtype=t, pin_memory=True)) for w, t, c in spec]
        for w, buf in sl["outs"]:
            _lib.check(L.fl_result_copy(res.handle, w, buf.data_ptr(),
                                        buf.numel() * buf.element_size(), _lib.MEM_HOST))
        return sz

    for sl in slots:  # warm-up (allocations, plan buffers, pinned outputs)
        issue(sl)
        drain(sl)
    K = max(depth + 1, args.e2e_steps)
    t0 = time.perf_counter()
    for k in range(K):
        issue(slots[k % depth])
        if k >= depth - 1:
            drain(slots[(k - depth + 1) % depth])
    for k in range(max(K - depth + 1, 0), K):
        drain(slots[k % depth])
    sec = (time.perf_counter() - t0) / K
    # single-call latency: one drop-in call at a time (upload -> assemble -> every
    # output downloaded), nothing overlapped -- what one solve_poisson caller sees
    singles = []
    for _ in range(3):
        t1 = time.perf_counter()
        issue(slots[0])
        drain(slots[0])
        singles.append(time.perf_counter() - t1)
    single = float(np.median(singles))
    h2d = h_nodes.numel() * 8 + h_elems.numel() * 4 + h_flags.numel() + (f_arr.nbytes if f_arr is not None else 0)
    d2h = sum(buf.numel() * buf.element_size() for _, buf in slots[0]["outs"])
    for sl in slots:
        L.fl_mesh_destroy(sl["mesh"])
        del sl["res"]
    return {"value": NT / sec, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": sec * 1e3, "steps": K,
            "single_call": {"value": NT / single, "unit": UNIT, "ms": single * 1e3, "calls": len(singles),
                            "timing": "median wall clock of one un-pipelined C-ABI call: H2D of the "
                                      "mesh arrays from pinned memory, fl_assemble, every output D2H"},
            "timing": (f"wall clock over {K} steps, {depth}-deep pipeline of fl_ctx "
                       "(upload | assemble | download overlap across consecutive steps), "
                       "host arrays in pinned memory")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cached", action="store_true", help="skip the cached-plan loop")
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--e2e-depth", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dump-gather", default=None,
                    help="N>1: gather the sharded A to rank 0 after the timed loop (NCCL send/recv) and save it")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per k_columns launch (from profiles/), echoed into roofline")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.warmup < 3:
        log("[bench] warning: fewer than 3 warm-up steps")
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.init_process_group(os.environ.get("FL_BENCH_BACKEND", "nccl"))
    if args.impl == "reference":
        run_reference_impl(args, rank, world)
        return
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
