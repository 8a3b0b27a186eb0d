#!/usr/bin/env python
"""Benchmark of the B200 FCS hot path (driver contract: one JSON line on rank 0).

Headline workload: BASELINE config 4 — dense FCS of a 1024^3 float32 tensor
(4 GiB, iid N(0,1), seeded device fill), J_n = 16384 (J~ = 49150), D = 4
families. A step is one K1 pass (st_fcs_dense) over the rank's slab of the
tensor (elements sharded by the last mode), plus — for N > 1 — the single NCCL
all-reduce of the D x J~ fp64 partials. value = tensor elements / s for the
whole job (strong scaling: the 1024^3 tensor is split across ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Also reported: roofline of K1 against the measured HBM copy bandwidth
(MEASURED_PEAKS.json), e2e through the host-buffer C-ABI call
(st_fcs_dense_host, pinned host tensor, H2D + compute + D2H inside the timed
region), the reference CPU path on a bounded sample (cpu_baseline), clocks
sampled during the timed region, and secondary lines for configs 2, 3, 5.
The input (4 GiB) is larger than L2 (126 MB), so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import ctypes as C
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

C4_DIMS = (1024, 1024, 1024)
C4_J, C4_D, C4_SEED = 16384, 4, 4
METRIC = "fcs_dense_tensor_elements_per_sec"
UNIT = "elements/s"
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def jt_of(dims, J):
    return len(dims) * J - len(dims) + 1


def algorithmic_bytes(elems, dims, D, J, esz=4):
    """tensor read once + D x sum(I) x 5 B tables + D x J~ x esz out."""
    return elems * esz + D * sum(dims) * 5 + D * jt_of(dims, J) * esz


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms (B200_PROFILING.md)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        busy = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        reasons = set()
        for s in busy:
            for bit, name in REASONS.items():
                if s[2] & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy),
                "sm_max_mhz": max(s[1] for s in busy), "reasons": sorted(reasons),
                "samples": len(busy)}


# --------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2106_13062_b200 as st
    from paper_2106_13062_b200 import _lib as L
    from paper_2106_13062_b200.dist import shard_range

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = L.lib()
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    dims = list(C4_DIMS)
    lo, hi = shard_range(dims[-1], rank, world)
    per_slab = dims[0] * dims[1]
    elems_local = per_slab * (hi - lo)
    jt = jt_of(dims, C4_J)

    # synthetic slab (device fill; see paper_2106_13062_b200/configs.py) and tables
    x = torch.empty(elems_local, dtype=torch.float32, device="cuda")
    L.check(lib.st_device_gaussian(L.ST_F32, C4_SEED ^ (rank << 32), elems_local,
                                   C.c_void_p(x.data_ptr()), sp))
    seeds = [st.family_seed(C4_SEED, d) for d in range(C4_D)]
    packed = torch.empty(C4_D * sum(dims), dtype=torch.int32, device="cuda")
    dims_a, lens_a = L.size_array(dims), L.size_array([C4_J] * 3)
    L.check(lib.st_family_tables(3, dims_a, lens_a, C4_D, L.u64_array(seeds),
                                 C.c_void_p(packed.data_ptr()), sp))
    out = torch.empty((C4_D, jt), dtype=torch.float64, device="cuda")
    ws_bytes = lib.st_fcs_dense_workspace(L.ST_F32, 3, dims_a, hi - lo, C4_D, lens_a)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")

    def sketch():
        L.check(lib.st_fcs_dense(L.ST_F32, C.c_void_p(x.data_ptr()), 3, dims_a, lo, hi - lo, C4_D,
                                 C.c_void_p(packed.data_ptr()), lens_a, C.c_void_p(out.data_ptr()),
                                 0, C.c_void_p(ws.data_ptr()), ws_bytes, sp))

    def step():
        sketch()
        if world > 1:
            dist.all_reduce(out, op=dist.ReduceOp.SUM)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # timed region: K steps, CUDA events on the launching stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            k_ev[i][0].record(stream)
            sketch()
            k_ev[i][1].record(stream)
            if world > 1:
                dist.all_reduce(out, op=dist.ReduceOp.SUM)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_ms = ev0.elapsed_time(ev1)
    k_ms = statistics.mean(a.elapsed_time(b) for a, b in k_ev)
    if world > 1:
        tt = torch.tensor([t_ms, k_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms, k_ms = float(tt[0]), float(tt[1])
    ms_per_step = t_ms / args.steps
    total_elems = int(np.prod(dims))
    value = total_elems / (ms_per_step * 1e-3)

    peak, peak_kind = hbm_peak()
    alg = algorithmic_bytes(elems_local, dims, C4_D, C4_J)
    achieved = alg / (k_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("c4_fcs_dense_fx_kernel_bytes_per_launch")
        except Exception:
            traffic = None

    # e2e: host-buffer C-ABI call (pinned host tensor; H2D + tables + K1 + D2H)
    e2e = None
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    host = torch.empty(elems_local, dtype=torch.float32, pin_memory=True)
    host.copy_(x)
    hout = np.empty((C4_D, jt), np.float64)
    seeds_a = L.u64_array(seeds)

    def e2e_call():
        L.check(lib.st_fcs_dense_host(L.ST_F32, C.c_void_p(host.data_ptr()), 3, dims_a, lo, hi - lo,
                                      C4_D, seeds_a, lens_a, hout.ctypes.data_as(C.c_void_p)))

    e2e_call()  # warm-up: device buffers are cached across calls
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
        if world > 1:
            tmp = torch.from_numpy(hout).cuda()
            dist.all_reduce(tmp)
            hout[:] = tmp.cpu().numpy()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt[0])
    e2e = {"value": total_elems / t_e2e, "unit": UNIT, "h2d_bytes_per_step": elems_local * 4,
           "d2h_bytes_per_step": C4_D * jt * 8, "ms_per_step": t_e2e * 1e3,
           "api": "st_fcs_dense_host (fcs_sketch(DenseTensor, HashFamily) x D)"}
    del host

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: seeded SplitMix64/Box-Muller N(0,1) device fill",
            "config": {"workload": "c4: dense FCS 1024x1024x1024 float32, J_n=16384 (J~=49150), "
                                   "D=4", "dims": dims, "hash_len": C4_J, "sketch_count": C4_D,
                       "composed_len": jt, "seed": C4_SEED, "parallelism": f"element-shard x{world} + nccl "
                                                         "allreduce" if world > 1 else "single",
                       "l2": "input 4 GiB > L2 126 MB: no flush needed"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind, "kernel_ms": k_ms,
                         "algorithmic_bytes_per_launch": alg,
                         "kernel": "fcs_dense_fx_kernel<8> (+ fx_sample_warps, fx_group, reduce_fx)"},
            "e2e": e2e,
            # per step: fx_sample_warps, fx_scale, fx_group (cached lookup), the scatter
            # fcs_dense_fx_kernel, its redo instantiation (exits unless flagged), reduce_fx
            "gpu_launches": 6 * args.steps,
            "clocks": clk.summary(),
        }
    if world == 1 and not args.no_secondary:
        try:
            line["secondary"] = secondary(x, cpu=not args.no_cpu)
        except Exception as e:  # never lose the headline
            line["secondary"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(threads=1, target_s=args.cpu_seconds)
        except Exception as e:
            line["cpu_baseline"] = {"error": repr(e)}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def fp64_peak():
    """Measured fp64 FMA peak (tools/microbench/peaks.cu -> profiles/fp64_peak.json)."""
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        with open(p) as f:
            return float(json.load(f)["fp64_fma_tflops"]), "measured (profiles/fp64_peak.json)"
    except Exception:
        return 37.0, "fallback (B200 nominal fp64)"


def fft_flops(M: int, transforms: int) -> float:
    """Nominal FLOPs of `transforms` real M-point FFTs (2.5 M log2 M each)."""
    import math
    return transforms * 2.5 * M * math.log2(M)


def roofline_hbm(alg_bytes: float, ms: float, peak: float) -> dict:
    ach = alg_bytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "algorithmic_bytes": alg_bytes}


def roofline_fp64(flops: float, ms: float, peak: float, kind: str) -> dict:
    ach = flops / (ms * 1e-3) / 1e12
    return {"bound": "fp64", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
            "frac": ach / peak, "flops": flops, "peak_kind": kind,
            "flop_model": "2.5 M log2 M per real M-point transform (5 N log2 N per complex N)"}


def median_time(fn, reps=5):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def secondary(x=None, cpu=True):
    """Configs 1, 2, 3, 5 on one GPU: device-resident inputs,
    preallocated outputs and workspaces, the C-ABI calls timed with CUDA
    events, median of >= 10 calls after warm-up. Each entry carries its
    roofline (HBM by algorithmic bytes; fp64 FFT rate for the spectral ones,
    against the measured DFMA peak) and the reference CPU path (oracle/_ref,
    one host thread) on the same inputs or a stated bounded sample. Also K1
    on the config-4 tensor for D = 1, 2, 4 and the fp64 K1 on 1024^3 (J =
    8192, D = 1)."""
    import ctypes as C

    import torch

    import paper_2106_13062_b200 as st
    from paper_2106_13062_b200 import _lib as L
    from paper_2106_13062_b200 import configs

    lib = L.lib()
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    peak, _ = hbm_peak()
    fpeak, fkind = fp64_peak()
    ref = None
    if cpu:
        from oracle import ref

    def median_ms(fn, reps=12):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        for a, b in evs:
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in evs)

    def dense_call(t, dims, fams, D, dtype):
        packed = st.packed_families(fams)
        lens = fams[0].hash_lens()
        out = torch.empty((D, fams[0].composed_len()), dtype=torch.float64, device="cuda")
        dims_a, lens_a = L.size_array(dims), L.size_array(lens)
        ws_bytes = lib.st_fcs_dense_workspace(dtype, len(dims), dims_a, dims[-1], D, lens_a)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")

        def call():
            L.check(lib.st_fcs_dense(dtype, C.c_void_p(t.data_ptr()), len(dims), dims_a, 0,
                                     dims[-1], D, C.c_void_p(packed.data_ptr()), lens_a,
                                     C.c_void_p(out.data_ptr()), 0, C.c_void_p(ws.data_ptr()),
                                     ws_bytes, sp))
        return call

    res = {}
    if x is not None:
        sweep = []
        for D in (1, 2, 4):
            fams = st.families_for(list(C4_DIMS), st.EstimatorConfig(C4_J, D, C4_SEED))
            ms = median_ms(dense_call(x, list(C4_DIMS), fams, D, L.ST_F32), 10)
            alg = algorithmic_bytes(x.numel(), C4_DIMS, D, C4_J)
            sweep.append({"D": D, "ms": ms, "elements_per_sec": x.numel() / (ms * 1e-3),
                          "hbm_frac": alg / (ms * 1e-3) / 1e9 / peak,
                          "updates_per_sec": D * x.numel() / (ms * 1e-3)})
        res["c4_family_sweep"] = sweep
        # fp64 K1 (64-bit fixed point) on the same geometry: 1024^3 fp64 (8 GiB), J = 8192, D = 1
        try:
            n = x.numel()
            x64 = torch.empty(n, dtype=torch.float64, device="cuda")
            L.check(lib.st_device_gaussian(L.ST_F64, 7, n, C.c_void_p(x64.data_ptr()), sp))
            fams = st.families_for(list(C4_DIMS), st.EstimatorConfig(8192, 1, 7))
            ms = median_ms(dense_call(x64, list(C4_DIMS), fams, 1, L.ST_F64), 5)
            alg = algorithmic_bytes(n, C4_DIMS, 1, 8192, esz=8)
            res["fp64_dense_1024^3_J8192_D1"] = {
                "ms": ms, "elements_per_sec": n / (ms * 1e-3),
                "roofline": roofline_hbm(alg, ms, peak),
                "kernel": "fcs_dense_fx64_kernel<32, full> (64-bit fixed point, two int32 ATOMS)"}
            del x64
            torch.cuda.empty_cache()
        except Exception as e:  # memory: 4 GiB fp32 + 8 GiB fp64 resident
            res["fp64_dense_1024^3_J8192_D1"] = {"error": repr(e)}

    # sparse (COO) FCS at config-4 geometry, 1 % density (north_star (1), O(nnz))
    try:
        nnz_t = (1 << 30) // 100
        g = torch.Generator(device="cuda").manual_seed(11)
        flat = torch.unique(torch.randint(0, 1 << 30, (nnz_t,), device="cuda", generator=g))
        nnz = flat.numel()
        coords = torch.stack([flat % 1024, (flat // 1024) % 1024, flat // (1 << 20)], dim=1)
        coords = coords.to(torch.int32).contiguous()
        vals = torch.randn(nnz, dtype=torch.float64, device="cuda", generator=g)
        fams = st.families_for(list(C4_DIMS), st.EstimatorConfig(C4_J, C4_D, C4_SEED))
        packed = st.packed_families(fams)
        dims_a, lens_a = L.size_array(list(C4_DIMS)), L.size_array([C4_J] * 3)
        outc = torch.empty((C4_D, jt_of(C4_DIMS, C4_J)), dtype=torch.float64, device="cuda")

        def coo_call():
            L.check(lib.st_fcs_coo(L.ST_F64, C.c_void_p(vals.data_ptr()),
                                   C.c_void_p(coords.data_ptr()), nnz, 3, dims_a, C4_D,
                                   C.c_void_p(packed.data_ptr()), lens_a,
                                   C.c_void_p(outc.data_ptr()), 0, None, sp))
        ms = median_ms(coo_call, 10)
        alg = nnz * (8 + 12) + C4_D * sum(C4_DIMS) * 5 + C4_D * jt_of(C4_DIMS, C4_J) * 8
        e = {"ms": ms, "nnz": nnz, "nnz_per_sec": nnz / (ms * 1e-3),
             "roofline": roofline_hbm(alg, ms, peak),
             "bound_note": "fp64 L2 reductions: nnz x D = %d RED.E.ADD.F64" % (nnz * C4_D)}
        if ref is not None:
            # the reference has no sparse type: a sparse tensor costs it the dense sweep
            # with the zero test (for_each_nonzero, sketch.cpp:48-61); sample: 16 slabs
            sample = np.zeros((1024, 1024, 16))
            fl = flat[flat < 16 * (1 << 20)].cpu().numpy()
            sample.reshape(-1, order="F")[fl] = vals[:fl.size].cpu().numpy()
            rt = ref.ResidentTensor.from_array(sample)
            tabs = [ref.hash_family(C4_DIMS, C4_J, ref.family_seed(C4_SEED, d))[:2]
                    for d in range(C4_D)]

            def ref_sparse():
                for b, s in tabs:
                    rt.fcs([b[0], b[1], b[2][:16]], [s[0], s[1], s[2][:16]], [C4_J] * 3)
            dt = median_time(ref_sparse, reps=3)
            rt.close()
            e["cpu_baseline"] = {"value": fl.size / dt, "unit": "nnz/s", "cores": 1,
                                 "kind": "reference",
                                 "sample": "16 of 1024 slabs (1024x1024x16, 1 % nonzero), D = 4: "
                                           "the reference's dense fcs_sketch with zero skipping "
                                           "(it has no sparse input), oracle/_ref, median of 3",
                                 "seconds": dt}
        res["c4_sparse_coo_1pct"] = e
        del flat, coords, vals
    except Exception as ex:
        res["c4_sparse_coo_1pct"] = {"error": repr(ex)}

    # c1: dense FCS of 100^3 fp64, D = 1 (the reference's CPU-runnable case)
    c = configs.C1
    x1 = configs.c1_tensor(c)
    t1 = torch.from_numpy(np.ascontiguousarray(x1.ravel(order="F"))).cuda()
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    ms = median_ms(dense_call(t1, list(c.dims), fams, c.sketch_count, L.ST_F64))
    e = {"ms": ms, "elements_per_sec": t1.numel() / (ms * 1e-3),
         "roofline": roofline_hbm(configs.algorithmic_bytes("c1"), ms, peak), "seed": c.seed,
         "note": "launch/latency-bound: 8 MB moves in 1.2 us at the HBM roofline"}
    if ref is not None:
        rt = ref.ResidentTensor.from_array(x1)
        b, s, _ = ref.hash_family(c.dims, c.hash_len, ref.family_seed(c.seed, 0))
        dt = median_time(lambda: rt.fcs(b, s, [c.hash_len] * 3))
        rt.close()
        e["cpu_baseline"] = {"value": t1.numel() / dt, "unit": UNIT, "cores": 1,
                             "kind": "reference",
                             "sample": "the whole c1 tensor: fcs_sketch(DenseTensor, family 0) "
                                       "via oracle/_ref, median of 5", "seconds": dt}
    res["c1_dense_fcs"] = e

    # c2: CP-form FCS, rank 50 400^3, D = 10
    c = configs.C2
    w, fs = configs.c2_cp(c)
    cp = st.CpTensor(w, fs)
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    packed = st.packed_families(fams)
    dims_a, lens_a = L.size_array(list(c.dims)), L.size_array(fams[0].hash_lens())
    out2 = torch.empty((c.sketch_count, fams[0].composed_len()), dtype=torch.float64,
                       device="cuda")
    ws2 = lib.st_fcs_cp_workspace(3, dims_a, cp.rank(), c.sketch_count, lens_a)
    wbuf2 = torch.empty(max(ws2, 1), dtype=torch.uint8, device="cuda")
    fptrs = (C.c_void_p * 3)(*[f.data_ptr() for f in cp._factors_cm])

    def cp_call():
        L.check(lib.st_fcs_cp(C.c_void_p(cp.weights.data_ptr()), cp.rank(), 3, dims_a, fptrs, 0,
                              cp.rank(), c.sketch_count, C.c_void_p(packed.data_ptr()), lens_a,
                              C.c_void_p(out2.data_ptr()), 0, C.c_void_p(wbuf2.data_ptr()), ws2,
                              sp))
    ms = median_ms(cp_call)
    M2 = 12288  # padded real length for J~ = 11998
    fl2 = fft_flops(M2, c.sketch_count * cp.rank() * 3 + c.sketch_count)
    e = {"ms": ms, "sketches_per_sec": c.sketch_count / (ms * 1e-3),
         "roofline": roofline_fp64(fl2, ms, fpeak, fkind),
         "roofline_hbm": roofline_hbm(configs.algorithmic_bytes("c2"), ms, peak),
         "seed": c.seed, "metric": "CP-FCS sketches/s (D=10 sketches of a rank-50 400^3 CP tensor)"}
    if ref is not None:
        nf = 2
        dt = median_time(lambda: [ref.fcs_cp(w, fs, c.hash_len, ref.family_seed(c.seed, d))
                                  for d in range(nf)], reps=1)
        e["cpu_baseline"] = {"value": nf / dt, "unit": "sketches/s", "cores": 1,
                             "kind": "reference",
                             "sample": f"{nf} of the 10 families: fcs_sketch(CpTensor) via "
                                       "oracle/_ref (FFTW absent: the shim's exact-length FFT)",
                             "seconds": dt}
    res["c2_cp_fcs"] = e

    # c3: one batched T(I,u,u) step (15 restarts x 10 families) and the full RTPM
    c = configs.C3
    t, lam, V = configs.c3_tensor(c)
    dt3 = st.DenseTensor.from_array(t)
    est = st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng = st.FcsEngine(dt3, est)  # warm-up (plans, pools)
    del eng
    torch.cuda.synchronize()
    ev0.record(stream)
    eng = st.FcsEngine(dt3, est)
    ev1.record(stream)
    torch.cuda.synchronize()
    build_ms = ev0.elapsed_time(ev1)
    Lr = configs.C3_INITS
    U = torch.randn(Lr, 200, dtype=torch.float64, device="cuda")
    Y = torch.empty((Lr, 200), dtype=torch.float64, device="cuda")
    z1 = torch.empty(Lr, dtype=torch.float64, device="cuda")

    def iuv_call(n=Lr):
        L.check(lib.st_engine_iuv(eng._h, n, C.c_void_p(U.data_ptr()),
                                  C.c_void_p(U.data_ptr()), 0, C.c_void_p(Y.data_ptr()), 1, sp))

    def uvw_call(n=Lr):
        L.check(lib.st_engine_uvw(eng._h, n, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()),
                                  C.c_void_p(U.data_ptr()), C.c_void_p(z1.data_ptr()), 1, sp))
    ms_iuv = median_ms(iuv_call, 20)
    ms_iuv1 = median_ms(lambda: iuv_call(1), 20)
    def pipelined_ms(fn, calls=100):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(calls):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / calls
    with ClockSampler(torch.cuda.current_device()) as clk3:
        pipe_iuv = pipelined_ms(iuv_call, 3000)  # >= 100 ms each: clock samples land inside
        pipe_iuv1 = pipelined_ms(lambda: iuv_call(1), 6000)
    ms_uvw = median_ms(uvw_call, 20)
    ms_uvw1 = median_ms(lambda: uvw_call(1), 20)
    # the same steps on the direct time-domain path (correlate.cu), which the
    # engine's cost rule does not pick at this geometry: the measured A/B
    eng.set_path("direct")
    ab = {"path_taken": "spectral (engine.cu use_direct cost rule)",
          "direct_iuv_step_pipelined_ms": pipelined_ms(iuv_call, 300),
          "direct_iuv_batch1_pipelined_ms": pipelined_ms(lambda: iuv_call(1), 300),
          "direct_uvw_step_pipelined_ms": pipelined_ms(uvw_call, 300)}
    eng.set_path("auto")
    ab["spectral_iuv_step_pipelined_ms"] = pipelined_ms(iuv_call, 300)
    ms_defl = median_ms(lambda: L.check(lib.st_engine_deflate(
        eng._h, C.c_double(0.0), C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()),
        C.c_void_p(U.data_ptr()), sp)), 10)
    rcfg = st.RtpmConfig(c.rank, Lr, configs.C3_ITERS, st.SketchBackend.FCS, est)
    st.rtpm(dt3, rcfg)  # warm-up: first launches of the driver's kernels, plans, pools
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cpd = st.rtpm(dt3, rcfg)
    torch.cuda.synchronize()
    t_rtpm = time.perf_counter() - t0
    R, T = c.rank, configs.C3_ITERS
    model = {"build_ms": build_ms, "restarts_ms": R * (T * ms_iuv + ms_uvw),
             "refinement_ms": R * (T * ms_iuv1 + ms_uvw1), "deflation_ms": R * ms_defl}
    model["sum_ms"] = sum(model.values())
    M3 = 9216  # padded real length for J~ = 8998
    fl3 = fft_flops(M3, 3 * Lr * c.sketch_count)
    e = {"iuv_step_ms": ms_iuv, "estimates_per_sec": Lr / (ms_iuv * 1e-3),
         "roofline": roofline_fp64(fl3, ms_iuv, fpeak, fkind),
         "roofline_hbm": roofline_hbm(1517680, ms_iuv, peak),
         "iuv_batch1_ms": ms_iuv1,
         "iuv_batch1_path": "8-CTA cluster per (vector, family) item, transposes over DSMEM, "
                            "median fused into the last cluster (spectral_cluster.cu)",
         "roofline_batch1": roofline_fp64(fft_flops(M3, 3 * c.sketch_count), ms_iuv1, fpeak, fkind),
         "pipelined_ms": {"iuv_step": pipe_iuv, "iuv_batch1": pipe_iuv1,
                          "note": "3000 / 6000 back-to-back calls on one stream (as inside rtpm)",
                          "clocks": clk3.summary()},
         "uvw_step_ms": ms_uvw, "uvw_batch1_ms": ms_uvw1,
         "deflate_ms": ms_defl, "rtpm_total_s": t_rtpm, "rtpm_timing": "second call (warm), host wall",
         "rtpm_breakdown_model": model, "estimator_paths_ab": ab, "seed": c.seed,
         "weights": [round(float(v), 6) for v in cpd.weights.cpu().numpy()]}
    if ref is not None:
        reng = ref.Engine(t, c.hash_len, c.sketch_count, c.seed)
        u0 = U[0].cpu().numpy()
        ncall = 8
        dt = median_time(lambda: [reng.iuu(u0) for _ in range(ncall)], reps=1)
        e["cpu_baseline"] = {"value": ncall / dt, "unit": "estimates/s", "cores": 1,
                             "kind": "reference",
                             "sample": f"{ncall} calls of the reference FcsEngine::iuu (each the "
                                       "median over D = 10 of T(I,u,u)) via oracle/_ref; FFTW "
                                       "absent: the shim's exact-length FFT", "seconds": dt}
        del reng
    res["c3_rtpm"] = e

    # c5: FCS of A (x) B, 512^2 operands, D = 8 (device-resident operands)
    c = configs.C5
    A, B = configs.c5_matrices(c)
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    packed5 = st.packed_families(fams)
    lens5 = L.size_array(fams[0].hash_lens())
    Ad = torch.from_numpy(np.ascontiguousarray(A.ravel(order="F"))).cuda()
    Bd = torch.from_numpy(np.ascontiguousarray(B.ravel(order="F"))).cuda()
    out5 = torch.empty((c.sketch_count, fams[0].composed_len()), dtype=torch.float64,
                       device="cuda")

    def kron_call():
        L.check(lib.st_fcs_kron(C.c_void_p(Ad.data_ptr()), 512, 512, C.c_void_p(Bd.data_ptr()),
                                512, 512, c.sketch_count, C.c_void_p(packed5.data_ptr()), lens5,
                                C.c_void_p(out5.data_ptr()), sp))
    ms = median_ms(kron_call)
    e = {"ms": ms, "sketches_per_sec": c.sketch_count / (ms * 1e-3),
         "roofline": roofline_hbm(configs.algorithmic_bytes("c5"), ms, peak), "seed": c.seed}
    if ref is not None:
        def ref_kron():
            for d in range(c.sketch_count):
                b, sg, _ = ref.hash_family(list(c.dims), c.hash_len, ref.family_seed(c.seed, d))
                fa = ref.fcs_dense_tables(A, [b[0], b[1]], [sg[0], sg[1]], [c.hash_len] * 2)
                fb = ref.fcs_dense_tables(B, [b[2], b[3]], [sg[2], sg[3]], [c.hash_len] * 2)
                ref.fft_convolve([fa, fb], len(fa) + len(fb) - 1)
        dt = median_time(ref_kron, reps=3)
        e["cpu_baseline"] = {"value": c.sketch_count / dt, "unit": "sketches/s", "cores": 1,
                             "kind": "reference",
                             "sample": "all 8 families: fcs_sketch of both operands + "
                                       "fft_convolve via oracle/_ref, median of 3",
                             "seconds": dt}
    res["c5_kron"] = e
    return res


# ------------------------------------------------------------ reference (CPU)
# Both CPU legs run the UNMODIFIED reference sources (oracle/_ref) and import
# nothing from paper_2106_13062_b200: the data come from the reference's own
# SplitMix64/next_gaussian (rng.cpp:8-21), rounded through float32 (config 4
# is fp32; the reference API is fp64-only, tensor.hpp:50-51), held in
# resident reference DenseTensors built outside the timed region.

def _host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class RefC4:
    """The config-4 workload on the reference: the 1024 i_3-slabs split into
    `nchunks` contiguous chunks (each a resident DenseTensor), D = 4 families
    (families_for(dims, {16384, 4, 4}), estimators.cpp:104-115). One pass =
    fcs_sketch of every (chunk, family) with the chunk's slice of the family's
    last-mode table (sharding by linearity), then the per-family
    sum of the chunk partials."""

    def __init__(self, slabs: int, nchunks: int, threads: int):
        import concurrent.futures as cf

        from oracle import ref
        self.ref = ref
        self.threads = max(1, threads)
        self.slabs = slabs
        nchunks = max(1, min(nchunks, slabs))
        bounds = [slabs * c // nchunks for c in range(nchunks + 1)]
        self.chunks = [(bounds[c], bounds[c + 1]) for c in range(nchunks)]
        self.fams = [ref.hash_family(C4_DIMS, C4_J, ref.family_seed(C4_SEED, d))[:2]
                     for d in range(C4_D)]

        def make(c):
            s0, s1 = self.chunks[c]
            return ref.ResidentTensor.gaussian(C4_SEED * 1000003 + s0, (1024, 1024, s1 - s0),
                                               round_f32=True)
        with cf.ThreadPoolExecutor(self.threads) as ex:
            self.tensors = list(ex.map(make, range(nchunks)))
        self.tasks = [(c, d) for c in range(nchunks) for d in range(C4_D)]
        self.jt = jt_of(C4_DIMS, C4_J)
        self.parts = np.zeros((len(self.tasks), self.jt))
        self.pool = cf.ThreadPoolExecutor(self.threads) if self.threads > 1 else None

    @property
    def elements(self) -> int:
        return C4_DIMS[0] * C4_DIMS[1] * self.slabs

    def _one(self, k):
        c, d = self.tasks[k]
        s0, s1 = self.chunks[c]
        b, s = self.fams[d]
        self.tensors[c].fcs([b[0], b[1], b[2][s0:s1]], [s[0], s[1], s[2][s0:s1]], [C4_J] * 3,
                            out=self.parts[k])

    def run(self) -> float:
        """One timed pass (wall clock, seconds); returns the elapsed time."""
        t0 = time.perf_counter()
        if self.pool is None:
            for k in range(len(self.tasks)):
                self._one(k)
        else:
            list(self.pool.map(self._one, range(len(self.tasks))))
        out = self.parts.reshape(len(self.chunks), C4_D, self.jt).sum(axis=0)
        dt = time.perf_counter() - t0
        assert out.shape == (C4_D, self.jt)
        return dt

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()
        for t in self.tensors:
            t.close()
        self.tensors = []


def cpu_baseline(threads: int = 1, target_s: float = 10.0):
    """The reference's own fcs_sketch(DenseTensor) (oracle/_ref) on a bounded
    sample of config 4: the first `slabs` i_3-slabs (1024 x 1024 x slabs),
    all D = 4 families, on `threads` host threads; median of 3 passes."""
    probe = RefC4(4, 1, threads)
    dt = probe.run()
    probe.close()
    slabs = int(min(256, max(4, target_s / 3.0 / max(dt, 1e-3) * 4)))
    w = RefC4(slabs, max(1, threads), threads)
    times = [w.run() for _ in range(3)]
    w.close()
    dt = statistics.median(times)
    return {"value": w.elements / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"1024x1024x{slabs} slab of config 4 ({w.elements} elements, fp32 values "
                      f"widened to fp64), D=4 families, reference fcs_sketch(DenseTensor) via "
                      f"oracle/_ref, median of 3",
            "seconds": dt}


def run_reference(args):
    """--impl reference: the reference CPU path on the FULL config-4 workload
    per step (2^30 elements, D = 4), every host core (harness-level split into
    slab chunks x families). Rank 0 only under torchrun."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    cores = _host_cores()
    w = RefC4(C4_DIMS[2], max(16, 2 * cores), cores)
    times = []
    for i in range(max(args.warmup, 0) + args.steps):
        dt = w.run()
        if i >= args.warmup:
            times.append(dt)
    w.close()
    ms = statistics.mean(times) * 1e3
    value = w.elements / (ms * 1e-3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded SplitMix64/Box-Muller N(0,1) (reference rng), fp32-rounded",
            "config": {"workload": "c4: dense FCS 1024x1024x1024 float32, J_n=16384 (J~=49150), "
                                   "D=4", "dims": list(C4_DIMS), "hash_len": C4_J,
                       "sketch_count": C4_D, "composed_len": jt_of(C4_DIMS, C4_J),
                       "seed": C4_SEED},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"the full workload per step: {len(w.chunks)} slab chunks "
                                       f"x {C4_D} families of fcs_sketch(DenseTensor) "
                                       "(oracle/_ref, unmodified reference sources), fp64"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_probe(args):
    """--probe (CPU test of the launcher): gloo all-reduce across the spawned
    ranks, rank 0 prints the world it saw."""
    import torch
    import torch.distributed as dist
    rank, world, _ = env_rank()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        seen = int(t.item())
        dist.destroy_process_group()
    else:
        seen = 1
    if rank == 0:
        print(json.dumps({"probe": True, "n_gpus": world, "ranks_seen": seen}), flush=True)


def spawn(args) -> int:
    """--gpus N > 1 without a torchrun environment: relaunch this script as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.probe:
        run_probe(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
