#!/usr/bin/env python
"""TT-embedding training-step benchmark (BASELINE.json metric).

One step = forward (lookup of the batch) + backward (core gradients) +
optimizer update of the cores, on the workload BASELINE.json names
(default: the papers100M-shaped config the north star's roofline target is
quoted on; --config selects another).  Inputs are seeded synthetic data of the
configs' shapes and distributions (paper_2206_10581_b200.synth).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config papers]
  python bench.py --impl reference ...   # the reference algorithm on host CPUs

N > 1 is launched by torchrun (one rank per GPU, NCCL): the global batch is
sharded by position, core gradients are all-reduced every step, and the
device time is the max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

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

METRIC = "TT-emb rows/sec fwd+bwd+update at 1/2/4/8 B200; % of FP32 peak; vs host-CPU ref"
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x20: "sync_boost", 0x40: "sw_thermal_slowdown", 0x80: "hw_thermal_slowdown",
           0x100: "hw_power_brake_slowdown", 0x200: "display_clock_setting"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="papers")
    p.add_argument("--seed", type=int, default=2026)
    p.add_argument("--path", default="auto", choices=["auto", "generic", "tc"])
    p.add_argument("--cpu-sample", type=int, default=0, help="rows per CPU-baseline step (0 = auto)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-tensor-path", action="store_true", help="skip the tensor-core path measurement")
    p.add_argument("--shard", default="owner", choices=["owner", "position"], help="N > 1 decomposition (dist.py)")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo: functional smoke test of the N > 1 path (ranks may share a GPU); not a measurement")
    p.add_argument("--graph", type=int, default=1, help="replay the step as one CUDA graph (1) or launch eagerly (0)")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi clocks and throttle reasons, sampled during the timed region."""

    def __init__(self, gpu_id: str):
        self.gpu_id, self.rows, self.proc = gpu_id, [], None

    def start(self):
        q = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for r in self.rows:
            parts = [x.strip() for x in r.split(",")]
            if len(parts) < 4:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[3], 16) if parts[3].startswith("0x") else int(parts[3])
            except ValueError:
                continue
            if bits & 0x1:  # idle sample, not under load
                continue
            sm.append(s)
            mx = m
            for b, name in REASONS.items():
                if bits & b:
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _traffic(config_name, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture (profiles/ncu_traffic.json), or None."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(config_name, {}).get(kernel)
    except (OSError, ValueError, AttributeError):
        return None


def level_costs(cfg):
    """c_l = N_{l-1} R_{l-1} n_l R_l MACs for levels l = 2..d (0-based k = 1..d-1)."""
    out, N = [], cfg.n[0]
    for k in range(1, cfg.d):
        out.append(N * cfg.R[k] * cfg.n[k] * cfg.R[k + 1])
        N *= cfg.n[k]
    return out


def algorithmic_flops(cfg, U):
    """Reuse-aware F = 6 sum_l U_l c_l (fwd 1 part, bwd 2 parts)."""
    return 6.0 * sum(u * c for u, c in zip(U[1:], level_costs(cfg)))


def _opt_kind(name):
    from paper_2206_10581_b200.config import WORKLOADS
    return WORKLOADS[name]["opt"]


def _size_sample(run, B, start, target_s, full_s):
    """Rows per CPU step: the full batch if a step over it is estimated to take
    <= full_s seconds, else grown from `start` until a step takes ~target_s
    (the multithreaded backward has a fixed per-call cost, so a one-point
    per-row estimate undershoots)."""
    S = min(B, start)
    while True:
        t0 = time.perf_counter()
        run(S)
        t = time.perf_counter() - t0
        if S >= B:
            return B
        if t * B / S <= full_s:
            return B
        if t >= 0.6 * target_s:
            return S
        S = int(min(B, S * min(8.0, target_s / max(t, 1e-6))))


def cpu_variant(cfg, name, idx, up, cores, f32, nthreads, rep_s=1.5, full_s=4.0, reps=5):
    """One CPU-baseline variant of BASELINE.md section 3: the oracle (the C
    restatement of the reference's lookup_batch / backward_lookup /
    apply_update, tt_embedding.cpp:110-125, autodiff.cpp:48-173) with fwd,
    bwd and the dense update timed separately (time.perf_counter, a steady
    clock), median of `reps` repetitions.  The rows per repetition are the full
    batch when a repetition is estimated to take <= full_s seconds, else the
    first S rows with S sized for ~rep_s seconds.  The value is MEASURED:
    S / (t_fwd + t_bwd + t_upd) of a real step over S rows (the update is the
    reference's dense update of every parameter, once per step) -- nothing is
    extrapolated."""
    import oracle
    B = len(idx)
    kind = {"sgd": oracle.SGD, "adagrad": oracle.ADAGRAD, "adam": oracle.ADAM}[_opt_kind(name)]
    if f32:
        cs = [np.ascontiguousarray(c, np.float32).copy() for c in cores]
        fwd, bwd, upd = oracle.lookup_batch_f32, oracle.backward_lookup_f32, oracle.apply_update_f32
        opt = oracle.OptState32(cfg, kind, 0.01)
    else:
        cs = [c.astype(np.float64) for c in cores]
        fwd, bwd, upd = oracle.lookup_batch, oracle.backward_lookup, oracle.apply_update
        opt = oracle.OptState(cfg, kind, 0.01)
    S = _size_sample(lambda n: (fwd(cfg, cs, idx[:n], nthreads), bwd(cfg, cs, idx[:n], up[:n], nthreads)),
                     B, 32 if max(cfg.R) >= 64 else 256, rep_s, full_s)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fwd(cfg, cs, idx[:S], nthreads)
        t1 = time.perf_counter()
        g, _ = bwd(cfg, cs, idx[:S], up[:S], nthreads)
        t2 = time.perf_counter()
        upd(cfg, cs, g, opt)
        t3 = time.perf_counter()
        times.append((t1 - t0, t2 - t1, t3 - t2))
    tf, tb, tu = (float(x) for x in np.median(np.array(times), axis=0))
    what = "fp32" if f32 else "fp64"
    rows = "the full batch" if S == B else f"the first {S} of {B} batch rows"
    return {"value": S / (tf + tb + tu), "unit": "rows/s", "cores": nthreads, "kind": "port",
            "sample": f"{what}, {nthreads} thread(s): fwd + bwd over {rows}, then the dense {_opt_kind(name)} "
                      f"update of all {sum(int(c.size) for c in cores)} params; each timed separately, "
                      f"median of {reps}; value = rows / (t_fwd + t_bwd + t_upd) of that measured step",
            "rows": S, "reps": reps, "ms": {"fwd": tf * 1e3, "bwd": tb * 1e3, "upd": tu * 1e3}}


def cpu_baseline(cfg, name, idx, up, cores):
    """BASELINE.md section 3's two variants on the host cores: (i) the faithful
    single-thread fp64 restatement and (ii) the multithreaded fp32 one over all
    host cores (rows split, fixed-order gradient reduction).  The line's value
    is (ii), the faster CPU number, in the arithmetic type the GPU path uses."""
    import oracle
    nt = oracle.num_threads()
    st = cpu_variant(cfg, name, idx, up, cores, False, 1)
    mt = cpu_variant(cfg, name, idx, up, cores, True, nt)
    out = {k: mt[k] for k in ("value", "unit", "cores", "kind", "sample")}
    out["variants"] = {"i_single_thread_fp64": st, "ii_multithread_fp32": mt}
    return out


def run_reference(a, rank):
    """--impl reference: the reference's CPU implementation of the path on the
    host cores.  The reference (tt_embedding.cpp, autodiff.cpp) needs Eigen,
    absent from this image, so its restatement in oracle/ runs: fp64 (the
    reference's arithmetic), OpenMP over every host core.  Each step is one
    real fwd + bwd + dense update over the first S rows of the workload's
    batch (S sized so a step takes ~2 s, so --steps K --warmup W ends within
    minutes); every step is timed and the line reports exactly what ran."""
    if rank != 0:
        return
    import oracle
    from paper_2206_10581_b200.config import workload_inputs, WORKLOADS
    name = a.config
    cfg, idx, up, cores = workload_inputs(name, a.seed)
    B = len(idx)
    nt = oracle.num_threads()
    kind = {"sgd": oracle.SGD, "adagrad": oracle.ADAGRAD, "adam": oracle.ADAM}[WORKLOADS[name]["opt"]]
    cs = [c.astype(np.float64) for c in cores]
    opt = oracle.OptState(cfg, kind, 0.01)
    S = a.cpu_sample or _size_sample(
        lambda n: (oracle.lookup_batch(cfg, cs, idx[:n], nt), oracle.backward_lookup(cfg, cs, idx[:n], up[:n], nt)),
        B, 64 if max(cfg.R) >= 64 else 512, 2.0, 4.0)

    def step():
        oracle.lookup_batch(cfg, cs, idx[:S], nt)
        g, _ = oracle.backward_lookup(cfg, cs, idx[:S], up[:S], nt)
        oracle.apply_update(cfg, cs, g, opt)

    for _ in range(a.warmup):
        step()
    per = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        step()
        per.append(time.perf_counter() - t0)
    tot = sum(per)
    v = S * a.steps / tot
    rows = "the full batch" if S == B else f"the first {S} of the {B}-row batch"
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "rows/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": tot / a.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "batch": B, "rows_per_step": S, "num_nodes": cfg.num_nodes,
                       "row_factors": cfg.m, "col_factors": cfg.n, "ranks": cfg.R,
                       "optimizer": WORKLOADS[name]["opt"]},
            "cpu_baseline": {"value": v, "unit": "rows/s", "cores": nt, "kind": "port",
                             "sample": f"each timed step: fwd + bwd over {rows} + the dense {WORKLOADS[name]['opt']} "
                                       f"update of all {sum(int(c.size) for c in cores)} params (fp64 restatement "
                                       f"of the reference, {nt} OpenMP threads); value = rows processed / measured "
                                       f"time of the {a.steps} timed steps"},
            "ms_per_step_each": [x * 1e3 for x in per],
            "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank)
        return
    import torch
    import torch.distributed as dist
    from paper_2206_10581_b200 import engine as E
    from paper_2206_10581_b200.config import WORKLOADS, workload_inputs
    from paper_2206_10581_b200.dist import DataParallelTT, OwnerShardedTT, shard_bounds

    if a.dist_backend == "gloo":
        # functional smoke test of the N > 1 code path on fewer GPUs than ranks:
        # host-side collectives, so no kernel waits on another rank; never a
        # measurement (the line says so)
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if a.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = a.config
    cfg, idx_all, up_all, cores = workload_inputs(name, a.seed)
    Bg = len(idx_all)
    lo, hi = shard_bounds(Bg, rank, world)
    B = hi - lo
    dev = torch.device("cuda", local)
    idx = torch.tensor(idx_all[lo:hi], device=dev)
    up = torch.tensor(up_all[lo:hi], device=dev)
    emb = E.TTEmbedding(cfg, local)
    emb.set_cores(cores)
    emb.set_path(a.path)
    opt = E.OptimizerState.make(cfg, getattr(E.OptKind, WORKLOADS[name]["opt"]), 0.01)
    emb.configure_optimizer(opt)
    dp = None
    if world > 1:
        dp = OwnerShardedTT(emb) if a.shard == "owner" else DataParallelTT(emb)
    out = torch.empty((B, cfg.emb_dim), dtype=torch.float32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    def step_eager():
        if dp is None:
            emb.forward(idx, out)
            emb.backward(up)
            emb.step()
        else:  # routing / all-reduce inside (dist.py)
            dp.forward(idx, out)
            dp.backward(up)
            dp.step()

    def timed(path):
        """Capture (world 1) and time `a.steps` steps on `path`; returns the
        max-over-ranks device time and the per-phase kernel times."""
        emb.set_path(path)
        step = step_eager
        graph, graph_kernels = None, 0
        if a.graph and world == 1:
            # capture forward + backward + update once (after a warm-up that sizes
            # every buffer) and replay it: one launch per step instead of ~60
            emb.snapshot_cores()
            step_eager()
            torch.cuda.synchronize()
            emb.sync()
            emb.restore_cores()
            s_cap = torch.cuda.Stream(device=dev)
            s_cap.wait_stream(torch.cuda.current_stream(dev))
            graph = torch.cuda.CUDAGraph()
            n0 = emb.launch_count()
            with torch.cuda.stream(s_cap):
                with torch.cuda.graph(graph, stream=s_cap):
                    step_eager()
            graph_kernels = emb.launch_count() - n0
            torch.cuda.current_stream(dev).wait_stream(s_cap)
            torch.cuda.synchronize()
            step = graph.replay
        # Every timed step starts from the same cores (restored outside the
        # timed events, like the L2 flush): repeated SGD steps on one fixed batch
        # diverge at the billion config (sum-gradients of Zipf-hot IDs), and a
        # rejected non-finite update would skip work.
        emb.snapshot_cores()
        for _ in range(a.warmup):
            emb.restore_cores()
            step()
        torch.cuda.synchronize()
        emb.sync()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        emb.profile_read()  # drop warm-up records
        emb.set_profiling(graph is None)
        l0 = emb.launch_count()
        for i in range(a.steps):
            emb.restore_cores()
            flush.zero_()
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
        launches = emb.launch_count() - l0
        if graph is not None:
            launches = graph_kernels * a.steps  # kernels replayed from the captured graph
        emb.set_profiling(False)
        prof = emb.profile_read()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        emb.sync()
        per_step = [s.elapsed_time(e) for s, e in ev]
        tt = torch.tensor([sum(per_step)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        if graph is not None:
            # per-phase kernel timing needs the eager launches (events on the
            # launching stream): the same K steps once more, eagerly
            emb.set_profiling(True)
            for i in range(a.steps):
                emb.restore_cores()
                flush.zero_()
                step_eager()
            torch.cuda.synchronize()
            emb.set_profiling(False)
            prof = emb.profile_read()
        emb.restore_cores()
        torch.cuda.synchronize()
        phase_ms = {k: (v[0] / v[1] if v[1] else 0.0) for k, v in prof.items()}
        return {"t_max": t_max, "per_step": per_step, "launches": launches, "phase_ms": phase_ms,
                "path": emb.last_path(), "graph": graph is not None,
                "kernels": {"fwd": emb.main_kernel(False), "bwd": emb.main_kernel(True)}}

    props = torch.cuda.get_device_properties(local)
    uuid = getattr(props, "uuid", None)
    sampler = ClockSampler(f"GPU-{uuid}" if uuid else str(local))
    sampler.start()
    time.sleep(0.3)
    main_run = timed(a.path)
    clocks = sampler.stop()
    U = emb.plan_stats()
    t_max, per_step, launches, graph_on = main_run["t_max"], main_run["per_step"], main_run["launches"], main_run["graph"]
    value = Bg * a.steps / (t_max / 1e3)
    ms_per_step = t_max / a.steps
    phase_ms = main_run["phase_ms"]
    path_used = main_run["path"]

    # the optional tensor-core path (tcgen05, BF16x3: fp32-level accuracy),
    # reported beside the FP32 FFMA headline (north star: "reported separately")
    tensor = None
    if a.path == "auto" and not a.no_tensor_path:
        tc_run = timed("tc")
        if tc_run["path"] == "fused-tc":
            tf_ = algorithmic_flops(cfg, U)
            tc_ms = tc_run["t_max"] / a.steps
            # dominant tensor kernel: k_tc_bwd (dG_F^T and dA on the tensor pipe,
            # dC on the CUDA cores) -- algorithmic FLOPs per launch as for the
            # FFMA kernel; the BF16x3 split issues 6 BF16 MMAs per algorithmic MAC
            # of its two products, compared with the measured dense BF16 peak
            costs_ = level_costs(cfg)
            uf_cf_ = U[-2] * costs_[-2] if len(costs_) >= 2 else 0
            ud_cd_ = U[-1] * costs_[-1]
            bwd_ms = tc_run["phase_ms"].get("bwd_main", 0.0)
            bwd_flops = 4.0 * uf_cf_ + 2.0 * ud_cd_
            mma_flops = 6.0 * 4.0 * uf_cf_
            peaks = {}
            try:
                peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            except (OSError, ValueError):
                pass
            bf16_peak = peaks.get("bf16_tflops")
            tensor = {"path": "fused-tc (tcgen05.mma kind::f16, BF16x3 six-product split, FP32 accumulate in TMEM)",
                      "value": Bg * a.steps / (tc_run["t_max"] / 1e3), "unit": "rows/s", "ms_per_step": tc_ms,
                      "ms_per_step_each": tc_run["per_step"], "phases_ms_per_step": tc_run["phase_ms"],
                      "tolerance": "|x - x_ref| <= 1e-5 a_ref (same bound as the FP32 path; tests/test_gpu_parity.py)",
                      "step_tflops": tf_ / (tc_ms * 1e-3) / 1e12,
                      "roofline": {
                          "bound": "tensor", "kernel": tc_run["kernels"]["bwd"] or "k_tc_bwd", "unit": "TFLOP/s",
                          "achieved": bwd_flops / (bwd_ms * 1e-3) / 1e12 if bwd_ms > 0 else None,
                          "bf16_mma_tflops": mma_flops / (bwd_ms * 1e-3) / 1e12 if bwd_ms > 0 else None,
                          "peak": bf16_peak, "peak_source": "MEASURED_PEAKS.json bf16_tflops (dense, burst)",
                          "frac": (bwd_flops / (bwd_ms * 1e-3) / 1e12 / bf16_peak) if (bwd_ms > 0 and bf16_peak) else None,
                          "issued_mma_frac": (mma_flops / (bwd_ms * 1e-3) / 1e12 / bf16_peak) if (bwd_ms > 0 and bf16_peak) else None,
                          "traffic": _traffic(name, tc_run["kernels"]["bwd"] or "k_tc_bwd"), "flops_per_launch": bwd_flops,
                          "ms_per_launch": bwd_ms,
                          "note": "frac = algorithmic FLOPs (4 U_F c_F + 2 U_d c_d) over the dense BF16 peak; "
                                  "issued_mma_frac = the BF16 MMA FLOPs actually issued (6 per algorithmic MAC of "
                                  "dG_F and dA, the BF16x3 split) over the same peak; "
                                  + ("the phase is k_fused_wdc (dC and the last core's W_u over the saved P_F, "
                                     "HBM-bound) + k_tc_bwd3 (dC staged by TMA, both dC operands in TMEM, bound by "
                                     "the CUDA cores' BF16x3 conversion), not by the tensor pipe (DESIGN.md c2)"
                                     if (tc_run["kernels"]["bwd"] or "") == "k_tc_bwd3" else
                                     "the kernel is bound by forming dC on the CUDA cores (latency of the per-ID "
                                     "loads), not by the tensor pipe (DESIGN.md c2)")},
                      "gpu_launches": tc_run["launches"]}
        emb.set_path(a.path)

    # roofline of the dominant kernel: its algorithmic FLOPs per launch over its
    # average launch duration, timed live with CUDA events on its stream
    flops = algorithmic_flops(cfg, U)
    peak = E.ffma_peak_tflops(local, 8192)
    peak_gemm = E.ffma_outer_tflops(local, 4096)
    costs = level_costs(cfg)
    fused = path_used.startswith("fused")
    # algorithmic FLOPs of the fused kernels (the last level's forward and W
    # run in the streaming kernels k_last_level / k_fused_w):
    #   k_fused_fwd = 2 U_F c_F;  k_fused_bwd = 4 U_F c_F (dG_F, dA) + 2 U_d c_d (dC pass)
    uf_cf = U[-2] * costs[-2] if len(costs) >= 2 else 0
    ud_cd = U[-1] * costs[-1]
    if fused:
        bwd_dom = phase_ms["bwd_main"] >= phase_ms["fwd_main"]
        dom = main_run["kernels"]["bwd" if bwd_dom else "fwd"] or ("k_fused_bwd" if bwd_dom else "k_fused_fwd")
        dom_flops = (4.0 * uf_cf + 2.0 * ud_cd) if bwd_dom else 2.0 * uf_cf
        dom_ms = phase_ms["bwd_main" if bwd_dom else "fwd_main"]
    else:
        dom, dom_flops, dom_ms = "whole step (generic path)", flops, ms_per_step
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12 if dom_ms > 0 else 0.0
    traffic = None
    prof_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_file):
        try:
            traffic = json.load(open(prof_file)).get(name, {}).get(dom)
        except (OSError, ValueError, AttributeError):
            traffic = None

    # e2e through the C-ABI with pinned host buffers (H2D inputs, D2H output rows)
    e2e = None
    if not a.no_e2e:
        h_idx = torch.tensor(idx_all[lo:hi]).pin_memory()
        h_up = torch.tensor(up_all[lo:hi]).pin_memory()
        h_out = torch.empty((B, cfg.emb_dim), dtype=torch.float32).pin_memory()
        lib = E.load_library()

        def e2e_sync_step():
            emb.restore_cores_on_engine_stream()
            E._raise(lib.tt_train_step_host(emb._h, h_idx.data_ptr(), B, h_up.data_ptr(), h_out.data_ptr()),
                     "tt_train_step_host")

        def e2e_run(n, depth=3):
            """n pipelined steps through tt_train_step_submit / _wait, up to `depth`
            in flight: later steps' uploads run under a step's compute and row
            download (the engine has three staging slots)."""
            inflight = 0
            for i in range(n):
                emb.restore_cores_on_engine_stream()
                emb.train_step_submit(h_idx, h_up, h_out)
                inflight += 1
                if inflight >= depth:
                    emb.train_step_wait()
                    inflight -= 1
            for _ in range(inflight):
                emb.train_step_wait()

        def e2e_step():
            if dp is None:
                e2e_sync_step()
            else:
                d_idx = h_idx.to(dev, non_blocking=True)
                d_up = h_up.to(dev, non_blocking=True)
                dp.forward(d_idx, out)
                h_out.copy_(out, non_blocking=True)
                dp.backward(d_up)
                dp.step()
                torch.cuda.synchronize()

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            e2e_step()
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_sync = Bg * a.steps / float(te.item())
        api = "tt_train_step_host (C-ABI)" if dp is None else f"TTEmbedding + {type(dp).__name__} (Python API)"
        value_e2e = e2e_sync
        if dp is None:  # the pipelined host-buffer API (the headline e2e when N = 1)
            e2e_run(2)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_run(a.steps)
            torch.cuda.synchronize()
            value_e2e = Bg * a.steps / (time.perf_counter() - t0)
            api = "tt_train_step_submit / tt_train_step_wait (C-ABI, up to three steps in flight)"
        e2e = {"value": value_e2e, "unit": "rows/s",
               "h2d_bytes_per_step": int(h_idx.numel() * 8 + h_up.numel() * 4),
               "d2h_bytes_per_step": int(h_out.numel() * 4),
               "api": api, "synchronous_value": e2e_sync,
               "synchronous_api": "tt_train_step_host (C-ABI)" if dp is None else api}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(cfg, name, idx_all, up_all, cores)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": name, "global_batch": Bg, "num_nodes": cfg.num_nodes, "row_factors": cfg.m,
                       "col_factors": cfg.n, "ranks": cfg.R, "optimizer": WORKLOADS[name]["opt"],
                       "parallelism": f"dp{world}", "path": path_used,
                       "shard": None if world == 1 else (
                           "owner: level-F core sharded by digit, IDs + upstream rows routed by all-to-all, small cores all-reduced"
                           if a.shard == "owner" else "position: batch by position, whole gradient buffer all-reduced"),
                       "cuda_graph": graph_on,
                       "l2": "256 MB buffer written between timed steps (outside the events)",
                       "cores": "restored from a device snapshot before every step (outside the events)",
                       "unique_per_level_rank0": U},
            "roofline": {"bound": "fp32", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak > 0 else None, "traffic": traffic,
                         "flops_per_launch": dom_flops, "ms_per_launch": dom_ms,
                         "peak_source": "FFMA microbenchmark (tt_ffma_peak_tflops) on this GPU, this run",
                         "gemm_shaped_ffma_tflops": peak_gemm,
                         "step_flops": flops, "step_tflops": flops / (ms_per_step * 1e-3) / 1e12,
                         "step_frac": flops / (ms_per_step * 1e-3) / 1e12 / peak if peak > 0 else None},
            "phases_ms_per_step": phase_ms,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "ms_per_step_each": per_step, "tensor_path": tensor,
        }
        if a.dist_backend == "gloo":
            line["data"] = "synthetic; gloo smoke run of the N > 1 code path (ranks may share a GPU): not a measurement"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
