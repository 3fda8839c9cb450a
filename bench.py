"""bench.py — CBIE fill + H-LU throughput on B200 (config 2 of BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl reference]

One step = one full pass of the hot path on the device with the geometry
resident in HBM: FAR/NEAR/SELF classification + near-field pair blocks (K1,
K3), H-matrix fill (dense leaves K2/K4, batched ACA K5, recompression K6) and
the H-LU factorisation (K7-K10).  metric = unknowns/s = N / (fill + H-LU time).
For N > 1 (torchrun) every rank factors its own replica of the problem
(weak scaling, no data-path collective); value = N * ranks / max step time.
Beside it, "fill_sharded" times the fill of ONE problem with its leaves sharded
over the ranks plus the NCCL exchange of the shards (strong scaling of the fill),
and "hlu_distributed" the block-row-distributed H-LU of that H-matrix.

--impl reference times the CPU oracle (numpy restatement of the reference,
oracle/) on a bounded sample of the same workload (see oracle/baseline.py).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# one hardware work queue per executor stream (see paper_2408_17116_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "CBIE H-matrix fill+H-LU throughput (unknowns/s)"
UNIT = "unknowns/s"


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _fp64_peak():
    """FP64 denominator: best probe of profiles/fp64_peak_r01.jsonl (cuBLAS ZGEMM/DGEMM
    8192^3 and a DFMA chain, measured on this pool's B200 by tools/fp64_peak.cu)."""
    best = 0.0
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.jsonl")) as f:
            for line in f:
                line = line.strip()
                if line.startswith("{"):
                    best = max(best, float(json.loads(line).get("tflops", 0.0)))
    except OSError:
        pass
    return (best, "measured (profiles/fp64_peak_r01.jsonl, cuBLAS ZGEMM 8192^3)") if best > 0 else \
        (37.0, "fallback (B200 FP64 nominal)")


def _ncu_traffic(kernel="k_trunc_gram"):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    ncu --set full capture (profiles/r01j_k_trunc_gram_ncu_raw.csv), or None."""
    import csv
    path = os.path.join(ROOT, "profiles", "r01j_k_trunc_gram_ncu_raw.csv")   # 280-problem launch
    try:
        rows = list(csv.reader(open(path)))
        h, units, v = rows[0], rows[1], rows[2]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(name)
            tot += float(v[i].replace(",", "")) * scale.get(units[i], 1.0)
        return tot
    except (OSError, ValueError, IndexError):
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _reduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_baseline_line(cfg: int, steps: int, warmup: int, level: int = 3):
    """The oracle (numpy port of the reference) on a bounded, projected sample of
    the same configuration (oracle/baseline.py)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import baseline
    for _ in range(warmup):
        baseline.step(cfg, level)
    n_tot, t_tot, det = 0, 0.0, {}
    for _ in range(steps):
        n, sec, det = baseline.step(cfg, level)
        n_tot += n
        t_tot += sec
    return n_tot / t_tot, t_tot / max(steps, 1), baseline.describe(cfg, level), det


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return 0
    v, sec, desc, det = cpu_baseline_line(args.config, args.steps, args.warmup, args.ref_level)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "config": {"workload": f"config{args.config}"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": desc,
                             "projection": det},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import numpy as np
    import torch
    rank, world, local = _dist()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2408_17116_b200 import _ffi, configs, geometry as geo
    from paper_2408_17116_b200 import hmatrix as hm
    from paper_2408_17116_b200.solver import build_hmatrix

    prob = configs.problem(args.config)
    prob.device = local
    gen = prob.generator()                       # geometry + tables resident in HBM
    lib = gen.dev.lib
    stream = torch.cuda.ExternalStream(gen.stream)
    N = prob.n_dofs

    def step():
        gen.classify()
        H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
        F = hm.hlu_factor(H, prob.effective_trunc_tol)
        return H, F

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    hstats, fstats = [], []
    l0 = lib.cbie_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            H, F = step()
            hstats.append(H.stats())
            fstats.append(F.stats())
            del H, F
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.cbie_launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    _barrier(world)
    ms = _reduce_max(ms, world)
    value = world * N / (ms / 1e3)

    # roofline: dominant kernel group = the H-LU recompressions (Gram-path / blocked
    # truncation kernels, trunc2.cu), FP64-bound; achieved = FP64 flops they executed
    # (counted on the device with the ranks they saw, SURVEY 8(d) convention) / their
    # CUDA-event time on the launching streams
    peaks, peak_src = _peaks()
    fp64_peak, fp64_src = _fp64_peak()
    tf = sum(f.get("flops_trunc2", 0.0) for f in fstats)
    tms = sum(f["trunc_kernel_ms"] for f in fstats)
    tl = sum(f["trunc_launches"] for f in fstats)
    tb = sum(f["trunc_alg_bytes"] for f in fstats)
    achieved = tf / (tms / 1e3) / 1e12 if tms > 0 else 0.0
    flops = sum(f["flops"] for f in fstats) / args.steps
    hlu_ms = statistics.mean(f["factor_device_ms"] for f in fstats)
    roof = {"bound": "tensor", "kernel": "H-LU recompression (k_trunc_gram + k_trunc2, FP64; "
            "B200 DMMA and DFMA share the FP64 peak)",
            "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
            "peak_source": fp64_src, "traffic": _ncu_traffic(),
            "traffic_source": "ncu --set full, one k_trunc_gram launch (profiles/r01j_k_trunc_gram_ncu_raw.csv, 280 problems)",
            "flops_per_launch": tf / max(tl, 1), "avg_launch_ms": tms / max(tl, 1),
            "share_of_step": tms / args.steps / ms,
            "share_note": "sum of per-launch event times over the concurrent recompression "
                          "streams / step time; > 1 means the launches overlap each other",
            "hbm_alg_bytes_per_launch": tb / max(tl, 1),
            "hlu_fp64_tflops": flops / (hlu_ms / 1e3) / 1e12,
            "hlu_fp64_frac": flops / (hlu_ms / 1e3) / 1e12 / fp64_peak}

    # N > 1: the fill of ONE problem sharded over the ranks (LPT leaf partition, no
    # collective during the fill) + the NCCL exchange of the shards (csrc/shard.cu);
    # max-over-ranks device time, reported beside the replica throughput
    fill_shard = hlu_dist = None
    if world > 1:
        from paper_2408_17116_b200 import dist as cdist
        cdist.init_nccl(gen, rank, world)
        HS = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol, shard=(rank, world, True))   # warm-up
        del HS
        t_f, t_x = [], []
        for _ in range(max(1, args.steps)):
            _barrier(world)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            HS = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol, shard=(rank, world, True))
            b.record(stream)
            torch.cuda.synchronize()
            t_f.append(a.elapsed_time(b))
            t_x.append(HS.stats().get("exchange_ms", 0.0))
        # block-row-distributed H-LU of that H-matrix (csrc/hlu_dist.cuh): ncclSend/Recv
        # of the blocks peers read between dependency levels, final broadcast of the factors
        try:
            FD = cdist.hlu_factor_distributed(HS, prob.effective_trunc_tol)   # warm-up
            del FD
            t_h = []
            for _ in range(max(1, args.steps)):
                _barrier(world)
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                FD = cdist.hlu_factor_distributed(HS, prob.effective_trunc_tol)
                b.record(stream)
                torch.cuda.synchronize()
                t_h.append(a.elapsed_time(b))
                dst = FD.stats()
                del FD
            h_ms = _reduce_max(statistics.median(t_h), world)
            hlu_dist = {"ms": h_ms, "single_gpu_hlu_ms": statistics.mean(f["factor_device_ms"] for f in fstats),
                        "xfer_bytes": dst.get("dist_xfer_bytes"), "final_bytes": dst.get("dist_final_bytes"),
                        "messages": dst.get("dist_msgs"), "row_level": dst.get("dist_row_level"),
                        "scheme": "block rows dealt cyclically, level-synchronous ncclSend/Recv of peer-read blocks"}
        except RuntimeError as exc:   # reported, not fatal for the replica / sharded-fill numbers
            hlu_dist = {"error": str(exc)[:200]}
        del HS
        f_ms = _reduce_max(statistics.median(t_f), world)
        x_ms = _reduce_max(statistics.median(t_x), world)
        single = statistics.mean(h["fill_ms"] for h in hstats)
        fill_shard = {"ms": f_ms, "exchange_ms": x_ms, "single_gpu_fill_ms": single,
                      "leaves": "LPT partition of the block-tree leaves, ncclBroadcast of the shards",
                      "speedup_vs_replica_fill": single / f_ms if f_ms > 0 else None}
        cdist.finalize(gen)

    # e2e through the public API with host buffers (geometry in, solution out)
    e2e = None
    if not args.no_e2e:
        import dataclasses
        t_e2e = []
        h2d = d2h = 0
        for it in range(max(3, min(args.steps, 5)) + 1):   # first iteration: one-off setup, not timed
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            H2, gen2, scaled2, _ = build_hmatrix(dataclasses.replace(prob))
            F2 = hm.hlu_factor(H2, prob.effective_trunc_tol)
            rhs = gen2.rhs(prob.excitation) * scaled2.row_scale
            x = F2.solve(rhs) * scaled2.col_scale
            b.record()
            torch.cuda.synchronize()
            if it > 0:                      # first call pays one-off library/context setup
                t_e2e.append(a.elapsed_time(b))
            smp, kind, par, star, coef = geo.device_arrays(prob.patches)
            h2d = smp.nbytes + kind.nbytes + par.nbytes + coef.nbytes + rhs.nbytes
            d2h = x.nbytes + 3 * gen2.pos.nbytes + gen2.sqrt_g.nbytes
            del H2, gen2, F2
        e_ms = _reduce_max(statistics.median(t_e2e), world)
        e2e = {"value": world * N / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "iter_ms": [round(t, 2) for t in t_e2e],
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "solver.build_hmatrix + hmatrix.hlu_factor + HLUFactors.solve (host arrays)"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": f"config{args.config}", "N": N, "patches": len(prob.patches),
                       "order": list(prob.patches[0].orders), "n_leaf": prob.n_leaf,
                       "eta": prob.eta, "aca_tol": prob.aca_tol,
                       "parallelism": f"replicas{world}" if world > 1 else "single",
                       "l2": "working set (H-matrix arena ~3.9 GB) >> 126 MB L2"},
            "gpu_launches": int(launches // args.steps), "roofline": roof,
            "phases_ms": {"fill": statistics.mean(h["fill_ms"] for h in hstats),
                          "hlu": statistics.mean(f["factor_device_ms"] for f in fstats)},
            "fp64_flops_per_step": flops,
            "fp64_flops_note": "H-LU FP64 flops executed on the device (gemm/trsm/getrf/recompression/"
                               "dense->LR, ranks as seen by the kernels); the fill is not counted",
            "compression_rate": hstats[-1]["compression_rate"],
            "clocks": clk.summary()}
    if e2e:
        line["e2e"] = e2e
    if fill_shard:
        line["fill_sharded"] = fill_shard
    if hlu_dist:
        line["hlu_distributed"] = hlu_dist
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sec, desc, det = cpu_baseline_line(args.config, 1, 0, args.ref_level)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": desc,
                                "projection": det}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-level", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
