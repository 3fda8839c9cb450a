"""bench.py — CBIE fill + H-LU throughput on B200 (BASELINE.json configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl reference]

Workload (N = 1): config 4 of BASELINE.json -- the seeded star-shaped PEC body,
N = 49,152 unknowns -- the largest configuration whose fill and H-LU fit one
B200 (config 5 does not).  One step = one full pass of the
hot path with the geometry resident in HBM: FAR/NEAR/SELF classification and
near-field pair blocks (K1, K3), H-matrix fill (dense leaves K2/K4, batched ACA
K5, recompression K6) and the H-LU factorisation (K7-K10).  metric =
unknowns/s = N / (fill + H-LU).  Config 2 (N = 12,288) is measured beside it
under "config2" (same step, same rules).

N > 1 (``--gpus N`` spawns the ranks itself via torch.distributed.run when it
is not already running under one): ONE problem per step, strong scaling --
the fill with its leaves sharded over the ranks plus the NCCL exchange of the
shards (csrc/shard.cu), then the block-row-distributed H-LU (csrc/hlu_dist.cuh);
value = N / max-over-ranks step time.

--impl reference times the CPU reference path on the box's host cores: the
oracle (numpy restatement of the reference, oracle/) on a bounded stratified
sample of the same configuration, projected to the whole run and calibrated
against the reference's own full run measured in the build container
(oracle/baseline.py, oracle/calibration.json).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# one hardware work queue per executor stream (see paper_2408_17116_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "CBIE H-matrix fill+H-LU throughput (unknowns/s)"
UNIT = "unknowns/s"
NCU_CAPTURE = os.path.join(ROOT, "profiles", "r02_k_trunc_gram_ncu_raw.csv")


def _dist():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _fp64_peak():
    """FP64 denominator: best probe of profiles/fp64_peak_r01.jsonl (cuBLAS ZGEMM/DGEMM
    8192^3 and a DFMA chain, measured on this pool's B200 by tools/fp64_peak.cu)."""
    best = 0.0
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.jsonl")) as f:
            for line in f:
                if line.strip().startswith("{"):
                    best = max(best, float(json.loads(line).get("tflops", 0.0)))
    except OSError:
        pass
    return (best, "measured (profiles/fp64_peak_r01.jsonl, cuBLAS ZGEMM 8192^3)") if best > 0 else \
        (37.0, "fallback (B200 FP64 nominal)")


def _ncu_capture():
    """(DRAM read + write bytes, algorithmic bytes, problems) of the committed
    `ncu --set full` capture of one k_trunc_gram launch, or Nones."""
    import csv
    try:
        rows = list(csv.reader(open(NCU_CAPTURE)))
        h, units, v = rows[0], rows[1], rows[2]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(name)
            tot += float(v[i].replace(",", "")) * scale.get(units[i], 1.0)
        meta = json.load(open(NCU_CAPTURE.replace("_ncu_raw.csv", "_launch.json")))
        return tot, meta.get("alg_bytes"), meta
    except (OSError, ValueError, IndexError):
        return None, None, None


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
            threading.Thread(target=self._read, daemon=True).start()
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
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


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


# --------------------------------------------------------------------------- CPU arm
def cpu_baseline(cfg: int):
    """The reference path on this host's cores: oracle port, bounded stratified sample,
    calibrated to the reference's measured full run (oracle/baseline.py)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import baseline
    n, sec, det = baseline.calibrated_step(cfg)
    return n / sec, sec, det


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return 0
    for _ in range(args.warmup if args.ref_warmup else 0):
        cpu_baseline(args.config)
    vals, secs, det = [], [], {}
    for _ in range(1 if args.ref_steps is None else args.ref_steps):   # one bounded sample (~2 min of CPU)
        v, sec, det = cpu_baseline(args.config)
        vals.append(v)
        secs.append(sec)
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": 0,
            "steps": len(vals), "warmup": args.warmup, "ms_per_step": statistics.median(secs) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "config": {"workload": f"config{args.config}"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                             "sample": det["sample"], "detail": det},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def measure_single(cfg: int, steps: int, warmup: int, local: int, clocks: bool = True):
    """Device-resident steps of one configuration on one GPU (fill + H-LU)."""
    import numpy as np
    import torch
    from paper_2408_17116_b200 import configs, hmatrix as hm

    prob = configs.problem(cfg)
    prob.device = local
    gen = prob.generator()                 # geometry + tables resident in HBM
    lib = gen.dev.lib
    stream = torch.cuda.ExternalStream(gen.stream)

    def step():
        gen.classify()
        H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol)
        F = hm.hlu_factor(H, prob.effective_trunc_tol)
        return H, F

    for _ in range(warmup):
        H, F = step()
        del H, F
    torch.cuda.synchronize()
    hstats, fstats = [], []
    l0 = lib.cbie_launch_count()
    e0, e1 = _events()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for i in range(steps):
            H, F = step()
            hstats.append(H.stats())
            fstats.append(F.stats())
            if i + 1 < steps:
                del H, F
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.cbie_launch_count() - l0
    ms = e0.elapsed_time(e1) / steps

    # accuracy of the timed factorisation: one solve with the last factors
    b = gen.rhs(prob.excitation) * gen.row_scale
    y = F.solve(b)
    res = float(np.linalg.norm(H.matvec(y) - b) / np.linalg.norm(b))
    ovf = max(f.get("trunc_overflow", 0) for f in fstats)
    del H, F

    # cold plan: the same step with the H-LU tape recorded from scratch (a new mesh or
    # frequency pays this once per factorisation)
    os.environ["CBIE_NO_PLAN_CACHE"] = "1"
    a, z = _events()
    a.record(stream)
    H, F = step()
    z.record(stream)
    torch.cuda.synchronize()
    cold = {"ms_per_step": a.elapsed_time(z), "record_ms": F.stats()["record_ms"],
            "hlu_device_ms": F.stats()["factor_device_ms"]}
    del os.environ["CBIE_NO_PLAN_CACHE"]
    del H, F
    return dict(prob=prob, gen=gen, ms=ms, hstats=hstats, fstats=fstats, launches=launches,
                clocks=clk.summary() if clocks else None, residual=res, overflow=ovf, cold=cold)


def roofline(m):
    """Dominant kernel family: the H-LU recompressions (k_trunc_gram, k_trunc2), FP64.
    achieved = FP64 flops they executed (counted on the device with the ranks they saw,
    SURVEY 8(d) convention) / their CUDA-event time on the launching streams."""
    fp64_peak, fp64_src = _fp64_peak()
    fs = m["fstats"]
    tf = sum(f.get("flops_trunc2", 0.0) for f in fs)
    tms = sum(f["trunc_kernel_ms"] for f in fs)
    tl = sum(f["trunc_launches"] for f in fs)
    tb = sum(f["trunc_alg_bytes"] for f in fs)
    steps = len(fs)
    achieved = tf / (tms / 1e3) / 1e12 if tms > 0 else 0.0
    flops = sum(f["flops"] for f in fs) / steps
    hlu_ms = statistics.mean(f["factor_device_ms"] for f in fs)
    traffic, cap_alg, meta = _ncu_capture()
    return {"bound": "fp64", "kernel": "H-LU recompression (k_trunc_gram + k_trunc2; FP64 DFMA, "
            "B200 DMMA and DFMA share the FP64 peak)",
            "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
            "peak_source": fp64_src,
            "traffic": traffic, "traffic_alg_bytes": cap_alg,
            "traffic_source": (f"ncu --set full of one k_trunc_gram launch ({os.path.basename(NCU_CAPTURE)}: "
                               f"{meta.get('problems')} problems, config {meta.get('config')}); "
                               "traffic_alg_bytes = that launch's own B_rc") if meta else None,
            "flops_per_launch": tf / max(tl, 1), "avg_launch_ms": tms / max(tl, 1),
            "share_of_step": tms / steps / m["ms"],
            "share_note": "sum of per-launch event times over the concurrent recompression "
                          "streams / step time; > 1 means the launches overlap each other",
            "hbm_alg_bytes_per_launch": tb / max(tl, 1),
            "hlu_fp64_tflops": flops / (hlu_ms / 1e3) / 1e12,
            "hlu_fp64_frac": flops / (hlu_ms / 1e3) / 1e12 / fp64_peak,
            "hlu_fp64_flops_per_step": flops}


def e2e_single(prob, iters: int):
    """The public API with host buffers: geometry in, H-matrix, H-LU, solve, solution out
    (solver.build_hmatrix + hmatrix.hlu_factor + HLUFactors.solve)."""
    import dataclasses
    import torch
    from paper_2408_17116_b200 import geometry as geo, hmatrix as hm
    from paper_2408_17116_b200.solver import build_hmatrix
    t_e2e, cold = [], None
    h2d = d2h = 0
    for it in range(iters + 2):
        if it == 1:                         # cold plan: the tape recorded inside the timed region
            os.environ["CBIE_NO_PLAN_CACHE"] = "1"
        torch.cuda.synchronize()
        a, b = _events()
        a.record()
        H2, gen2, scaled2, _ = build_hmatrix(dataclasses.replace(prob))
        F2 = hm.hlu_factor(H2, prob.effective_trunc_tol)
        rhs = gen2.rhs(prob.excitation) * scaled2.row_scale
        x = F2.solve(rhs) * scaled2.col_scale
        b.record()
        torch.cuda.synchronize()
        os.environ.pop("CBIE_NO_PLAN_CACHE", None)
        if it == 1:
            cold = a.elapsed_time(b)
        elif it > 1:                        # it 0 pays one-off library/context setup
            t_e2e.append(a.elapsed_time(b))
        smp, kind, par, star, coef = geo.device_arrays(prob.patches)
        h2d = smp.nbytes + kind.nbytes + par.nbytes + coef.nbytes + rhs.nbytes + \
            (star.nbytes if star is not None else 0)
        d2h = x.nbytes + 3 * gen2.pos.nbytes + gen2.sqrt_g.nbytes
        del H2, gen2, F2
    return t_e2e, cold, h2d, d2h


def run_single(args):
    import torch
    local = 0
    torch.cuda.set_device(local)
    N_cfg = {}
    m = measure_single(args.config, args.steps, args.warmup, local)
    prob = m["prob"]
    N = prob.n_dofs
    value = N / (m["ms"] / 1e3)
    hs, fs = m["hstats"], m["fstats"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": m["ms"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": f"config{args.config}", "N": N, "patches": len(prob.patches),
                       "order": list(prob.patches[0].orders), "n_leaf": prob.n_leaf, "eta": prob.eta,
                       "aca_tol": prob.aca_tol, "parallelism": "single",
                       "l2": "inputs larger than L2 (H-matrix + factor arena >> 126 MB)"},
            "gpu_launches": int(m["launches"] // args.steps), "roofline": roofline(m),
            "phases_ms": {"fill": statistics.mean(h["fill_ms"] for h in hs),
                          "hlu": statistics.mean(f["factor_device_ms"] for f in fs)},
            "plan": {"warm_record_ms": statistics.mean(f["record_ms"] for f in fs),
                     "cold_step_ms": m["cold"]["ms_per_step"], "cold_record_ms": m["cold"]["record_ms"],
                     "cold_value": N / (m["cold"]["ms_per_step"] / 1e3),
                     "note": "timed steps reuse the recorded H-LU tape of the block structure "
                             "(same mesh); cold = one step with the tape recorded from scratch"},
            "accuracy": {"residual": m["residual"], "residual_bound": 100 * prob.aca_tol,
                         "trunc_overflow": m["overflow"]},
            "compression_rate": hs[-1]["compression_rate"], "clocks": m["clocks"]}
    del m
    if not args.no_e2e:
        t_e2e, cold, h2d, d2h = e2e_single(prob, max(3, min(args.steps, 5)))
        e_ms = statistics.median(t_e2e)
        line["e2e"] = {"value": N / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
                       "iter_ms": [round(t, 2) for t in t_e2e], "cold_plan_ms": cold,
                       "cold_plan_value": N / (cold / 1e3),
                       "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                       "api": "solver.build_hmatrix + hmatrix.hlu_factor + HLUFactors.solve "
                              "(host arrays); cold_plan: the H-LU tape recorded inside the timed call"}
    if args.config != 2 and not args.no_secondary:
        m2 = measure_single(2, 5, 3, local, clocks=False)
        line["config2"] = {"value": m2["prob"].n_dofs / (m2["ms"] / 1e3), "ms_per_step": m2["ms"],
                           "N": m2["prob"].n_dofs, "steps": 5, "warmup": 3,
                           "phases_ms": {"fill": statistics.mean(h["fill_ms"] for h in m2["hstats"]),
                                         "hlu": statistics.mean(f["factor_device_ms"] for f in m2["fstats"])},
                           "cold_step_ms": m2["cold"]["ms_per_step"],
                           "residual": m2["residual"], "trunc_overflow": m2["overflow"],
                           "roofline_frac": roofline(m2)["frac"]}
        del m2
    if not args.no_cpu:
        v, sec, det = cpu_baseline(args.config)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": det["sample"], "detail": det}
    print(json.dumps(line), flush=True)
    acc = line["accuracy"]
    if acc["trunc_overflow"] or not acc["residual"] <= acc["residual_bound"]:
        print(f"accuracy check failed: {acc}", file=sys.stderr)
        return 3
    return 0


def run_multi(args):
    """N > 1: one problem per step -- sharded fill + NCCL shard exchange, then the
    block-row-distributed H-LU; max-over-ranks device time (strong scaling)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    rank, world, local = _dist()
    assert world == args.gpus, f"WORLD_SIZE {world} != --gpus {args.gpus}"
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2408_17116_b200 import configs, dist as cdist, hmatrix as hm
    prob = configs.problem(args.config)
    prob.device = local
    gen = prob.generator()
    lib = gen.dev.lib
    stream = torch.cuda.ExternalStream(gen.stream)
    cdist.init_nccl(gen, rank, world)
    N = prob.n_dofs

    def step():
        gen.classify()
        H = hm.HMatrix(gen, prob.n_leaf, prob.eta, prob.aca_tol, shard=(rank, world, True))
        F = cdist.hlu_factor_distributed(H, prob.effective_trunc_tol)
        return H, F

    for _ in range(args.warmup):
        H, F = step()
        del H, F
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    l0 = lib.cbie_launch_count()
    hs, fs = [], []
    e0, e1 = _events()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for i in range(args.steps):
            H, F = step()
            hs.append(H.stats())
            fs.append(F.stats())
            if i + 1 < args.steps:
                del H, F
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.cbie_launch_count() - l0
    ms = _reduce_max(e0.elapsed_time(e1) / args.steps, world)
    b = gen.rhs(prob.excitation) * gen.row_scale
    res = float(np.linalg.norm(H.matvec(F.solve(b)) - b) / np.linalg.norm(b))
    line = {"metric": METRIC, "value": N / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": f"config{args.config}", "N": N, "n_leaf": prob.n_leaf,
                       "eta": prob.eta, "aca_tol": prob.aca_tol,
                       "parallelism": f"leaf-sharded fill + block-row H-LU over {world} GPUs",
                       "l2": "inputs larger than L2"},
            "gpu_launches": int(launches // args.steps),
            "phases_ms": {"fill": _reduce_max(statistics.mean(h["fill_ms"] for h in hs), world),
                          "exchange": _reduce_max(statistics.mean(h.get("exchange_ms", 0.0) for h in hs), world),
                          "hlu": _reduce_max(statistics.mean(f["factor_device_ms"] for f in fs), world)},
            "hlu_distributed": {"xfer_bytes": fs[-1].get("dist_xfer_bytes"),
                                "final_bytes": fs[-1].get("dist_final_bytes"),
                                "messages": fs[-1].get("dist_msgs"), "row_level": fs[-1].get("dist_row_level")},
            "accuracy": {"residual": res, "residual_bound": 100 * prob.aca_tol},
            "clocks": clk.summary()}
    del H, F
    cdist.finalize(gen)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def spawn(args):
    """--gpus N outside torchrun: launch N ranks on this node (127.0.0.1 rendezvous)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-steps", type=int, default=None, help="reference arm: steps (default --steps)")
    ap.add_argument("--ref-warmup", action="store_true", help="reference arm: run the warm-up steps too")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    rank, world, _ = _dist()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.impl == "reference":
        return run_reference(args)
    if world > 1:
        return run_multi(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
