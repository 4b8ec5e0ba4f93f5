#!/usr/bin/env python3
"""Benchmark of the HPS-multigrid hot path (BASELINE.json metric).

A step is one pass of the hot path over one synthetic BASELINE config:
element ItI build -> skeleton assembly -> level merges -> MG preconditioner
-> preconditioned FGMRES solve.  Headline `value` = preconditioned-GMRES
DOF-iterations/s (skeleton DOF x FGMRES iterations / device solve time, inputs
resident in HBM); `setup` = HPS setup elements/s (n^2 / device setup time).
`e2e` = the same GMRES metric through the public C ABI with host buffers
(pinned rhs H2D + solve + x D2H inside the timed region).

  python bench.py [--config 3] [--steps K] [--warmup W] [--gpus N] [--impl b200|reference]

Default: BASELINE cfg3 (128 x 128 elements, N = 20, kappa = 400; 1.24 M
skeleton DOF, 14 merge levels) -- the largest single-RHS config, where both
BASELINE targets (setup vs FP64 peak, GMRES vs HBM) are defined; cfg4 (32
right-hand sides) is the second documented line (--config 4).

Multi-GPU (torchrun): the config is sharded by quadtree subtree over the
ranks (NCCL: owner-computes top merges with send / recv of box maps at
setup; distributed Krylov vectors with allreduced inner products and
global-row exchanges in the matvec and the V-cycle; cfg4's 32 right-hand
sides too), value = the problem's DOF-iterations / max-over-ranks time,
scaling "strong"; --replicas runs independent copies instead ("weak").
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

def fp64_peak() -> dict:
    """Measured FP64 tensor-core (DMMA) peak of this pool's B200s: the
    sustained figure (4 s back to back, clocks sampled) from the committed
    probe record, else the round-1 burst probe."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")) as f:
            d = json.load(f)
        return {"tflops": d["dmma_sustained_tflops"], "burst": d["dmma_burst_tflops"],
                "source": "profiles/r02_fp64_peak.json (DMMA m8n8k4, 4 s back to back, sustained)"}
    except (OSError, KeyError, ValueError):
        return {"tflops": 37.1, "burst": 37.1,
                "source": "profiles/r01_fp64_peak_probe.log (DMMA burst)"}


FP64 = fp64_peak()
FP64_DMMA_PEAK_TFLOPS = FP64["tflops"]
KAPPA = [10.0, 40.0, 160.0, 400.0, 600.0]
SHAPE = {0: (4, 8), 1: (16, 16), 2: (64, 16), 3: (128, 20), 4: (256, 12)}
RESTART = [50, 50, 100, 100, 60]
TOL = [1e-10, 1e-10, 1e-10, 1e-10, 1e-8]
METRIC = "precond GMRES DOF-iterations/s"
UNIT = "DOF-iterations/s"


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if s[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def gmres_roofline(state, its, restart, solve_s, hbm_gbs) -> dict:
    """Pinned bytes of all timed iterations: operators + fused
    CGS2 vector traffic 16 dim (4(j+1)+6) at Arnoldi step j.  Multi-RHS
    (cfg4): FP64 bound: 8 R flops per stored operator entry per
    block iteration, against the measured DMMA peak."""
    R = state.get("nrhs", 1)
    if R > 1:
        flops = sum(8.0 * R * state["pinned_bytes"] / 16.0 * b for b in state["timed_block_its"])
        achieved = flops / solve_s / 1e12
        return {"pinned_flops_per_block_iteration": 8.0 * R * state["pinned_bytes"] / 16.0,
                "block_iterations": state["timed_block_its"], "nrhs": R, "achieved": achieved,
                "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s (fp64)",
                "frac": achieved / FP64_DMMA_PEAK_TFLOPS}
    total = 0.0
    for n_it in its:
        for i in range(n_it):
            j = i % restart
            total += state["pinned_bytes"] + 16.0 * state["dim"] * (4 * (j + 1) + 6)
    achieved = total / solve_s / 1e9
    return {"pinned_bytes_per_iteration_operators": state["pinned_bytes"],
            "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s", "frac": achieved / hbm_gbs}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def config_dict(config: int, seed: int, world: int, sharded: bool) -> dict:
    """The workload description, identical in both arms (same_config)."""
    n, N = SHAPE[config]
    L = 2 * (n.bit_length() - 1)
    return {"workload": f"cfg{config}", "n": n, "N": N, "kappa": KAPPA[config],
            "dof": 4 * n * (n - 1) * (N - 1), "elements": n * n,
            "nrhs": 32 if config == 4 else 1, "levels": L, "restart": RESTART[config],
            "tol": TOL[config], "seed": seed, "mg": "depth=L, gamma=1, coarse_iters=4",
            "krylov": "fgmres, reorthogonalize=true (driver.cpp:125-132)",
            "l2": "flushed between steps (256 MB)",
            "parallelism": (f"quadtree-subtree sharding x{world} (NCCL)" if sharded
                            else f"replicas x{world}")}


# ---------------------------------------------------------------- CPU side
# The reference C++ needs Eigen3 (absent on this image and the GPU box), so
# the CPU side is the oracle/ restatement of the reference algorithm (same
# block-map layout, partial-pivot LUs, MGS+reorth FGMRES), kind "port".
def oracle_setup(config: int, seed: int, threads: int, n: int = 0, kappa: float = 0.0):
    """Full setup as the reference driver times it (driver.cpp:41-51,138-171):
    elements + skeleton + hierarchy + preconditioner."""
    from oracle import pyoracle
    # T / H only per element: the reference keeps each element's dense t x t
    # operator and LU for the solution recovery (element.hpp:61-106), 160 GB
    # at cfg3 -- not timed here, and beyond the host's memory
    pyoracle.set_lean_elements(True)
    smp = pyoracle.sample(2, config=config, seed=seed, n=n)
    t0 = time.perf_counter()
    S = pyoracle.Session.from_sample(smp, kappa or KAPPA[config], threads=threads)
    S.build_hierarchy(0, False)
    depth = 2 * (smp["n"].bit_length() - 1)
    S.precond(depth=depth, gamma=1, coarse_iters=4)
    return S, time.perf_counter() - t0, smp["n"] ** 2


def oracle_iterations(S, restart: int, tol: float, max_iters: int) -> tuple[int, float]:
    """FGMRES (MGS + reorthogonalisation, record_history off: driver.cpp:125-132)
    from the zero guess, at most max_iters iterations; (iterations, seconds)."""
    _, rep = S.solve(S.rhs(), True, restart=restart, tol=tol, max_iters=max_iters, reorth=True,
                     record_history=False)
    return rep["iterations"], rep["seconds"]


def cpu_baseline_sample(config: int, seed: int) -> dict:
    """Bounded CPU sample for the b200 line (rank 0, N = 1, ~10-30 s, one
    thread as the reference runs): config's element order N and kappa h on a
    16 x 16 patch of elements (cfg <= 1: the config itself), full setup and
    FGMRES solve with the oracle."""
    n_cfg, N = SHAPE[config]
    n = min(16, n_cfg)
    kappa = KAPPA[config] * n / n_cfg
    S, t_setup, ne = oracle_setup(config, seed, 1, n=n, kappa=kappa)
    its, secs = oracle_iterations(S, RESTART[config], TOL[config], 2000)
    dim = S.dim
    S.close()
    sample = (f"oracle restatement, 1 thread: cfg{config}'s elements (N={N}, kappa h="
              f"{KAPPA[config] / n_cfg:.4g}) on a {n}x{n} patch, full setup + FGMRES "
              f"({its} iterations)" if n < n_cfg else
              f"oracle restatement, 1 thread: full cfg{config} setup + FGMRES ({its} iterations)")
    return {"value": dim * its / secs, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample,
            "setup_elements_per_s": ne / t_setup}


def run_reference(args, rank, world):
    """--impl reference: the CPU reference algorithm on all host threads, on
    the b200 arm's config.  The setup runs once and is timed whole (the
    HPS-setup metric); each step is then a bounded sample of the solve: FGMRES
    from the zero guess for min(its, k) iterations on the built hierarchy
    (k sized so a step takes ~10 s)."""
    if rank != 0:
        return  # rank 0 alone runs the reference on the host cores
    threads = os.cpu_count() or 1
    S, t_setup, ne = oracle_setup(args.config, args.seed, threads)
    restart, tol = RESTART[args.config], TOL[args.config]
    # size the sample: one iteration's cost, then ~10 s per step
    it1, s1 = oracle_iterations(S, restart, tol, 1)
    k = max(1, min(2000, int(10.0 / max(s1, 1e-3))))
    for _ in range(args.warmup):
        oracle_iterations(S, restart, tol, k)
    dof_its, solve_s, its = 0, 0.0, []
    for _ in range(args.steps):
        it, sec = oracle_iterations(S, restart, tol, k)
        dof_its += S.dim * it
        solve_s += sec
        its.append(it)
    value = dof_its / solve_s
    sample = (f"full cfg{args.config} setup once (timed: {t_setup:.1f} s), then each step = "
              f"FGMRES from the zero guess for at most {k} iterations on that hierarchy "
              f"(oracle restatement, {threads} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * solve_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic", "config": config_dict(args.config, args.seed, world, False),
        "iterations": its,
        "setup": {"metric": "HPS setup elements/s", "value": ne / t_setup,
                  "ms_per_step": 1e3 * t_setup},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "setup_elements_per_s": ne / t_setup},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    S.close()
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU side
def run_b200(args, rank, world, local):
    import numpy as np
    import torch
    import paper_2511_00735_b200 as hps

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prob = hps.problem(2, args.config, seed=args.seed)
    ctx = hps.Context(local)
    if world > 1 and not args.replicas:
        # Quadtree-subtree sharding of ONE problem over the ranks (NCCL).
        uid = [hps.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        ctx.attach_nccl(uid[0], rank, world)
    ne = prob.n ** 2
    coeff_d = torch.from_numpy(np.ascontiguousarray(prob.coeff)).cuda(local)
    src_d = torch.from_numpy(np.ascontiguousarray(prob.source).view(np.float64)).cuda(local)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")
    restart, tol = prob.restart, prob.tol
    state = {}

    verbose = bool(os.environ.get("HPSB_BENCH_VERBOSE"))

    def step(profile: bool = False):
        import ctypes
        ctx.timer_start()
        w0 = time.perf_counter()
        h = ctypes.c_void_p()
        hps._check(hps._lib.hpsb_elements_build_dev(
            ctx._h, prob.n, prob.order, prob.eta, ctypes.c_void_p(coeff_d.data_ptr()),
            None if prob.source_zero else ctypes.c_void_p(src_d.data_ptr()), ctypes.byref(h)))
        el = hps.ElementRecords(ctx, h, prob.n, prob.order, prob.eta)
        w1 = time.perf_counter()
        sk = hps.assemble_skeleton(el, prob)
        w2 = time.perf_counter()
        hier = hps.build_hierarchy(sk, factor_coarse=False)
        w3 = time.perf_counter()
        pc = hps.build_preconditioner(hier, coarse_iters=4)
        t_setup = ctx.timer_stop()
        w4 = time.perf_counter()
        if verbose:
            print(f"[setup wall ms] elements {1e3 * (w1 - w0):.1f} skeleton {1e3 * (w2 - w1):.1f} "
                  f"hierarchy {1e3 * (w3 - w2):.1f} (device {1e3 * hier.build_seconds:.1f}) "
                  f"precond {1e3 * (w4 - w3):.1f}", file=sys.stderr)
        cfg = hps.KrylovConfig(restart, tol, 2000, 0, 1)
        nrhs = sk.nrhs
        x = torch.empty(2 * sk.dim * nrhs, dtype=torch.float64, device=f"cuda:{local}")
        if nrhs > 1:
            # cfg4: all right-hand sides in lockstep, one multi-RHS operator
            # pass per iteration (hpsb_fgmres_batch_dev)
            reps = (hps.SolveReport * nrhs)()
            hps._check(hps._lib.hpsb_fgmres_batch_dev(
                sk._h, pc._h, ctypes.c_void_p(sk.rhs_dev_ptr(0)), ctypes.c_void_p(x.data_ptr()),
                nrhs, cfg, reps), allow=(hps.OK,))
            seconds, it_total = reps[0].seconds, sum(r.iterations for r in reps)
            state["block_its"] = state.get("block_its", []) + [max(r.iterations for r in reps)]
        else:
            rep = hps.SolveReport()
            hps._check(hps._lib.hpsb_fgmres_dev(sk._h, pc._h, ctypes.c_void_p(sk.rhs_dev_ptr(0)),
                                                ctypes.c_void_p(x.data_ptr()), cfg,
                                                ctypes.byref(rep)), allow=(hps.OK,))
            seconds, it_total = rep.seconds, rep.iterations
        fe, fm = hier.pinned_flops()
        state.update(dim=sk.dim, pc_bytes=pc.bytes_per_apply, depth=hier.depth, nrhs=nrhs,
                     pinned_flops=fe + fm, pinned_bytes=pc.pinned_bytes_per_iteration)
        return t_setup, seconds, it_total, sk.dim

    def flush_l2():
        flush.zero_()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 0)):
        step()
        flush_l2()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    setup_s = solve_s = 0.0
    dof_its = 0
    its = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            ts, tv, it, dim = step()
            setup_s += ts
            solve_s += tv
            dof_its += dim * it
            its.append(it)
            if state.get("nrhs", 1) > 1:
                state.setdefault("timed_block_its", []).append(state["block_its"][-1])
            flush_l2()
    torch.cuda.synchronize()
    launches = ctx.launches - launches0
    sharded = world > 1 and not args.replicas
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([setup_s, solve_s, dof_its, ne * args.steps], dtype=torch.float64,
                         device=f"cuda:{local}")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        setup_max, solve_max = mx[0].item(), mx[1].item()
        if sharded:  # one problem solved by all ranks together
            dof_total, elem_total = dof_its, ne * args.steps
        else:        # independent replicas
            dof_total, elem_total = sm[2].item(), sm[3].item()
    else:
        setup_max, solve_max, dof_total, elem_total = setup_s, solve_s, dof_its, ne * args.steps
    value = dof_total / solve_max
    setup_value = elem_total / setup_max

    # ---- per-kernel roofline from one profiled (untimed) step
    ctx.profile_reset()
    ctx.profile(True)
    step()
    ctx.profile(False)
    prof = ctx.profile_entries()
    peaks = measured_peaks()
    # dominant kernel: the multi-RHS V-cycle runs the same kernels under two
    # direction labels (vcycle_up_batch / vcycle_down_batch): one entry
    fam = dict(prof)
    ub, db = fam.pop("vcycle_up_batch", None), fam.pop("vcycle_down_batch", None)
    if ub or db:
        parts = [x for x in (ub, db) if x]
        fam["vcycle_batch"] = {k: sum(x[k] for x in parts) for k in ("launches", "ms", "bytes", "flops")}
    dom = max(fam.items(), key=lambda kv: kv[1]["ms"])
    name, d = dom
    if d["flops"] > 0 and d["bytes"] == 0 or name in ("element_iti", "zgemm_dmma", "vcycle_batch"):  # multi-RHS apply: FP64 bound
        achieved = d["flops"] / (d["ms"] * 1e-3) / 1e12
        roof = {"kernel": name, "bound": "tensor", "achieved": achieved,
                "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s (fp64)",
                "frac": achieved / FP64_DMMA_PEAK_TFLOPS, "traffic": None,
                "peak_source": FP64["source"]}
    else:
        achieved = d["bytes"] / (d["ms"] * 1e-3) / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    roof["launches"] = d["launches"]
    # DRAM traffic per launch of the same kernel label from a committed ncu
    # capture of this config (profiles/r02_traffic.json, else r01), when there is one
    try:
        ent = {}
        for fn in ("r02_traffic.json", "r01_traffic.json"):
            pth = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", fn)
            if os.path.exists(pth):
                ent = json.load(open(pth)).get(f"cfg{args.config}", {})
                if name in ent:
                    break
        if name in ent:
            roof["traffic"] = ent[name]
            roof["traffic_unit"] = "bytes per launch (DRAM read + write, ncu)"
            roof["traffic_source"] = ent.get("source", "")
            roof["algorithmic_bytes_per_launch"] = d["bytes"] / max(d["launches"], 1)
    except (OSError, ValueError):
        pass
    kernels = {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                   "GBps": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1),
                   "TFLOPs": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3)}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}

    # ---- e2e through the public ABI with host buffers (rhs H2D, x D2H)
    el_h = hps.build_elements(ctx, prob)
    sk_h = hps.assemble_skeleton(el_h, prob)
    hier_h = hps.build_hierarchy(sk_h, factor_coarse=False)
    pc_h = hps.build_preconditioner(hier_h, coarse_iters=4)
    nrhs_e = state.get("nrhs", 1)
    rhs_np = np.stack([sk_h.rhs(b) for b in range(nrhs_e)]) if nrhs_e > 1 else sk_h.rhs()
    rhs_host = torch.from_numpy(rhs_np).pin_memory().numpy()
    e2e_dof, e2e_t = 0, 0.0
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        if nrhs_e > 1:
            x, reps_e = hps.fgmres_batch(sk_h, rhs_host, pc_h, restart=restart, tol=tol)
            its_e = sum(r["iterations"] for r in reps_e)
        else:
            x, rep = hps.fgmres(sk_h, rhs_host, pc_h, restart=restart, tol=tol)
            its_e = rep["iterations"]
        e2e_t += time.perf_counter() - t0
        e2e_dof += sk_h.dim * its_e
    e2e_value = e2e_dof / e2e_t
    # e2e setup: host coefficient arrays -> preconditioner ready (previous
    # objects released first, as in the timed steps)
    del pc_h, hier_h, sk_h, el_h
    import gc
    gc.collect()
    ctx.synchronize()
    t0 = time.perf_counter()
    el2 = hps.build_elements(ctx, prob)
    sk2 = hps.assemble_skeleton(el2, prob)
    hier2 = hps.build_hierarchy(sk2, factor_coarse=False)
    hps.build_preconditioner(hier2, coarse_iters=4)
    e2e_setup = ne / (time.perf_counter() - t0)

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * (setup_max + solve_max) / args.steps,
        "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": config_dict(args.config, args.seed, world, sharded),
        "iterations": its,
        "setup": {"metric": "HPS setup elements/s", "value": setup_value,
                  "ms_per_step": 1e3 * setup_max / args.steps},
        "solve_ms_per_step": 1e3 * solve_max / args.steps,
        "precond_bytes_per_apply": state["pc_bytes"],
        # Path-level rooflines with SURVEY §8(d)'s pinned numerators (one rank's
        # share when sharded): setup flops vs the measured FP64 DMMA peak, and
        # per-iteration operator + CGS2 vector bytes vs the measured HBM copy rate.
        "roofline_setup": {
            "pinned_flops": state["pinned_flops"],
            "achieved": state["pinned_flops"] * args.steps / setup_max / 1e12,
            "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s (fp64)",
            "frac": state["pinned_flops"] * args.steps / setup_max / 1e12 / FP64_DMMA_PEAK_TFLOPS},
        "roofline_gmres": gmres_roofline(state, its, restart, solve_max, peaks["hbm_gbs"]),
        "roofline": roof,
        "kernels": kernels,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": 16 * state["dim"] * state.get("nrhs", 1),
                "d2h_bytes_per_step": 16 * state["dim"] * state.get("nrhs", 1),
                "setup_elements_per_s": e2e_setup},
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(args.config, args.seed)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas instead of subtree sharding")
    args = ap.parse_args()
    if args.seed is None:
        args.seed = args.config
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
