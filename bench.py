#!/usr/bin/env python
"""bench.py — throughput of the PFEM explicit-FE hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--no-extras]

Workload: BASELINE.json config 3 — unit cube, 64^3 nodes, Kuhn T4
(1,500,282 tets), compressible Neo-Hookean mu=0.4 lambda=0.6, S=4 displacement fields,
fp32.  One STEP = one pass of §8 rows a2-a6 over the batch: the fused
energy+residual kernel (pfem_energy with W_e and r) followed by the matrix-free tangent
K(u).v (pfem_tangent_apply) on the same 4 fields.  value = element-samples per second
(E*S per step / step time), whole job over all ranks.  Inputs rotate over 3 independent
copies (mesh + fields, ~0.5 GB) so every step reads HBM, not L2 (no flush in the timed
region).  Row a7 (warm-started CG, config 4) and config 5 are reported under "extras".

--impl reference times the CPU oracle (oracle/, fp64) on a bounded sample of the same
workload on this box's host cores (the reference arm of this tier).
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

METRIC = "element-samples/s through fused energy+residual and K(u)v (config 3)"
UNIT = "element-samples/s"
N_COPIES = 3


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- bytes model
# FMA-pipe slots per element-sample of the 3-D Neo-Hookean kernels (counted from
# the formulas of element.cuh; the compiled phase 1 issues exactly these, 338 / 488 packed
# FFMA2-class instructions per element for 4 samples)
FMA_SLOTS_ER_NH3 = 169
FMA_SLOTS_KV_NH3 = 244


def bytes_energy_residual(E, N, d, S, s, want_W=True, mat_per_elem=0, K=1):
    """Algorithmic bytes of one fused energy+residual launch: conn, grad, vol,
    material read once; u read once; r written once; W_e written once; totals."""
    return (E * ((d + 1) * 4 + (d * d + 1) * s + mat_per_elem * s) +
            S * (N * d * s * 2 + (E * s if want_W else 0)) + S * K * s)


def bytes_tangent(E, N, d, S, s, nh, mat_per_elem=0, masked=False):
    """K(u).v: element arrays once; v read, Kv written, u read (NH), mask read (1 B/DOF)."""
    return (E * ((d + 1) * 4 + (d * d + 1) * s + mat_per_elem * s) +
            S * N * d * s * (3 if nh else 2) + (N * d if masked else 0))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


# ----------------------------------------------------------------------------- GPU arm
def build_workload(torch, pf, dev, prob, copies):
    """`copies` independent (mesh, material, u, v, outputs) sets on the device."""
    sets = []
    rng = np.random.default_rng(3005)
    v_host = rng.standard_normal(prob.u.shape)
    for _ in range(copies):
        mesh = pf.Mesh(torch.as_tensor(prob.coords, device=dev), torch.as_tensor(prob.conn, device=dev),
                       dtype=torch.float32)
        mat = pf.Material(prob.model, prob.param_kind,
                          torch.as_tensor(np.asarray(prob.p0), dtype=torch.float32, device=dev),
                          torch.as_tensor(np.asarray(prob.p1), dtype=torch.float32, device=dev))
        u = torch.as_tensor(prob.u, dtype=torch.float32, device=dev).contiguous()
        v = torch.as_tensor(v_host, dtype=torch.float32, device=dev).contiguous()
        S = u.shape[0]
        outs = (torch.empty((S, 1), dtype=torch.float32, device=dev),
                torch.empty((S, prob.n_elems), dtype=torch.float32, device=dev),
                torch.empty_like(u))
        Kv = torch.empty_like(u)
        mesh.workspace(S)
        sets.append({"mesh": mesh, "mat": mat, "u": u, "v": v, "outs": outs, "Kv": Kv})
    return sets


def step(pf, st, ev=None):
    if ev is not None:
        ev[0].record()
    pf.energy(st["mesh"], st["mat"], st["u"], elem_energy=True, residual=True, out=st["outs"])
    if ev is not None:
        ev[1].record()
    pf.tangent_apply(st["mesh"], st["mat"], st["v"], u=st["u"], out=st["Kv"])
    if ev is not None:
        ev[2].record()


def run_gpu(args):
    import torch
    import torch.distributed as tdist
    import paper_2601_03086_b200 as pf
    from pfem_gen import config3

    world, rank, local = dist_info()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)
    pf.load()
    # weak scaling: every rank owns its own batch of 4 fields on the (replicated) mesh
    prob = config3(seed_base=3000 + 1000 * rank) if rank else config3()
    E, N, d, S = prob.n_elems, prob.n_nodes, prob.dim, prob.n_samples
    t_prep0 = time.perf_counter()
    sets = build_workload(torch, pf, dev, prob, N_COPIES)
    torch.cuda.synchronize()
    prep_s = (time.perf_counter() - t_prep0) / N_COPIES

    for i in range(args.warmup):
        step(pf, sets[i % N_COPIES])
    torch.cuda.synchronize()

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    # the sampler needs ~0.2 s to start: keep the GPU busy with untimed steps meanwhile (an idle
    # GPU drops its clocks, and the first timed steps would then run during the ramp-up; with
    # the driver's 20 timed steps that inflated the per-kernel averages by ~5%)
    t_spin, i_spin = time.perf_counter(), 0
    while time.perf_counter() - t_spin < 0.2:
        step(pf, sets[i_spin % N_COPIES])
        i_spin += 1
        if i_spin % 16 == 0:
            torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    pf.launch_count(reset=True)
    t_start.record()
    for i in range(K):
        step(pf, sets[i % N_COPIES], evs[i])
    t_end.record()
    torch.cuda.synchronize()
    launches = pf.launch_count()
    if world > 1:
        tdist.barrier()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    er_ms = np.array([e[0].elapsed_time(e[1]) for e in evs])
    tg_ms = np.array([e[1].elapsed_time(e[2]) for e in evs])
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / K
    value = world * E * S / (ms_per_step * 1e-3)

    peak, peak_src = load_peaks()
    B_er = bytes_energy_residual(E, N, d, S, 4)
    B_tg = bytes_tangent(E, N, d, S, 4, nh=True)
    er_avg = float(er_ms.mean())
    traffic = load_traffic().get("config3_energy_residual")
    roofline = {"bound": "hbm", "achieved": B_er / (er_avg * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": B_er / (er_avg * 1e-3) / 1e9 / peak,
                "traffic": None if traffic is None else traffic.get("dram_bytes_per_launch"),
                "kernel": "k_assemble<3,NH,f32,ENERGY_RESIDUAL,ST=4> (pfem_energy)",
                "algorithmic_bytes": B_er, "avg_launch_us": er_avg * 1e3, "median_launch_us": float(np.median(er_ms)) * 1e3,
                "min_launch_us": float(er_ms.min()) * 1e3, "peak_source": peak_src,
                "tangent": {"kernel": "k_assemble<3,NH,f32,TANGENT,ST=4> (pfem_tangent_apply)",
                            "algorithmic_bytes": B_tg, "avg_launch_us": float(tg_ms.mean()) * 1e3,
                            "median_launch_us": float(np.median(tg_ms)) * 1e3, "min_launch_us": float(tg_ms.min()) * 1e3,
                            "achieved": B_tg / (tg_ms.mean() * 1e-3) / 1e9,
                            "frac": B_tg / (tg_ms.mean() * 1e-3) / 1e9 / peak}}

    # ALU view of the same two kernels (config 3 sits past the FP32 ridge).  One
    # FMA-pipe slot = one lane's FFMA / FMUL / FADD (packed FFMA2 = two slots per lane and issue);
    # slots per element-sample as the arithmetic of element.cuh is written, peak =
    # the FFMA2 rate measured now by pfem_fma_peak (outside the timed region).
    try:
        pk2, pk1, pk64 = pf.fma_peak("ffma2"), pf.fma_peak("ffma"), pf.fma_peak("dfma")
        alu = {"unit": "T lane-FMA slots/s", "peak": pk2 / 1e12, "peak_ffma": pk1 / 1e12, "peak_dfma": pk64 / 1e12,
               "peak_source": "pfem_fma_peak (dependent FFMA2 / FFMA / DFMA chains, measured in this run)"}
        for key, ops, ms in (("energy_residual", FMA_SLOTS_ER_NH3, er_avg), ("tangent", FMA_SLOTS_KV_NH3, float(tg_ms.mean()))):
            ach = ops * E * S / (ms * 1e-3)
            alu[key] = {"slots_per_element_sample": ops, "achieved": ach / 1e12, "frac": ach / pk2,
                        "floor_us": ops * E * S / pk2 * 1e6}
        roofline["alu"] = alu
        roofline["note"] = ("bound 'hbm' is the roofline the north star grades; by arithmetic config 3 sits past the "
                            "FP32 ridge: the FMA-pipe floors (alu.*.floor_us, measured peak) exceed the HBM times "
                            f"({B_er / peak / 1e3:.1f} / {B_tg / peak / 1e3:.1f} us)")
    except Exception as exc:   # a diagnostic: the bench line stands without it
        roofline["alu"] = {"error": str(exc)}

    # ---------------- e2e: host buffers through the public API, copies inside the timed region.
    # Every step copies its inputs (u, v) from pinned host memory and its results (totals, r,
    # K.v) back; the copies run on their own streams (H2D and D2H are full duplex on PCIe) and
    # overlap the neighbouring steps' compute through two device buffer sets (events order
    # each set's reuse), so the step rate is bounded by the slowest of the three.
    ss = [sets[0], sets[1 % N_COPIES]]
    u_h = ss[0]["u"].cpu().pin_memory()
    v_h = ss[0]["v"].cpu().pin_memory()
    outs_h = [(torch.empty(ss[0]["outs"][0].shape, dtype=torch.float32).pin_memory(),
               torch.empty(ss[0]["outs"][1].shape, dtype=torch.float32).pin_memory(),
               torch.empty(ss[0]["u"].shape, dtype=torch.float32).pin_memory(),
               torch.empty(ss[0]["u"].shape, dtype=torch.float32).pin_memory()) for _ in range(2)]
    tot_h, w_h, r_h, kv_h = outs_h[0]
    Ke = max(20, min(50, K))   # enough steps that the three-stream pipeline's fill and drain do not dominate
    cur = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]        # inputs of set i landed
    ev_used = [torch.cuda.Event() for _ in range(2)]      # compute of set i done (inputs free, outputs ready)
    ev_back = [torch.cuda.Event() for _ in range(2)]      # outputs of set i copied to the host
    for i in range(2):
        for e in (ev_used[i], ev_back[i]):
            e.record(cur)

    def e2e_step(k):
        i = k % 2
        sti = ss[i]
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_used[i])
            sti["u"].copy_(u_h, non_blocking=True)
            sti["v"].copy_(v_h, non_blocking=True)
            ev_in[i].record(s_in)
        cur.wait_event(ev_in[i])
        cur.wait_event(ev_back[i])
        step(pf, sti)
        ev_used[i].record(cur)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_used[i])
            th, wh, rh, kh = outs_h[i]
            th.copy_(sti["outs"][0], non_blocking=True)
            wh.copy_(sti["outs"][1], non_blocking=True)
            rh.copy_(sti["outs"][2], non_blocking=True)
            kh.copy_(sti["Kv"], non_blocking=True)
            ev_back[i].record(s_out)

    for k in range(4):
        e2e_step(k)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    s_in.wait_stream(cur)    # the first copies start after the opening event
    s_out.wait_stream(cur)
    for k in range(Ke):
        e2e_step(k)
    cur.wait_stream(s_out)   # the last results are on the host before the closing event
    cur.wait_stream(s_in)
    b.record(cur)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / Ke
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": world * E * S / (e2e_ms * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": int(u_h.numel() * 4 + v_h.numel() * 4),
           "d2h_bytes_per_step": int((tot_h.numel() + w_h.numel() + r_h.numel() + kv_h.numel()) * 4),
           "d2h_tensors": "totals [S,1], W_e [S,E], residual [S,N,3], K(u)v [S,N,3]",
           "ms_per_step": e2e_ms, "overlap": "H2D / compute / D2H on 3 streams, 2 buffer sets"}

    extras = {}
    if rank == 0 and not args.no_extras:
        del sets
        torch.cuda.empty_cache()
        extras = run_extras(torch, pf, dev, peak)
        extras["config3_prepare_s"] = prep_s
    # every kernel the north star grades (>= 60% of the HBM roofline on the >= 1M-element
    # configs), in the line itself so the driver's parse keeps them
    graded = {"config3_energy_residual": {"us": roofline["avg_launch_us"], "frac": roofline["frac"],
                                          "algorithmic_bytes": B_er},
              "config3_Kv": {"us": roofline["tangent"]["avg_launch_us"], "frac": roofline["tangent"]["frac"],
                             "algorithmic_bytes": B_tg}}
    for k in ("config4_Kv", "config5_energy_residual"):
        if k in extras:
            graded[k] = {"us": extras[k]["us"], "frac": extras[k]["frac"],
                         "algorithmic_bytes": extras[k]["algorithmic_bytes"]}
    roofline["graded"] = graded

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
           "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded generators, pfem_gen)",
           "config": {"workload": "config3", "mesh": "unit cube 64^3 nodes, Kuhn T4", "n_elems": E, "n_nodes": N,
                      "model": "neohookean mu=0.4 lam=0.6", "samples_per_rank": S, "global_batch": S * world,
                      "step": "pfem_energy(W_e, totals, residual) + pfem_tangent_apply(K(u)v)",
                      "assembly": "csr", "parallelism": f"replicas x{world} (independent batches, no collective)",
                      "spin_up": "untimed steps for 0.2 s while the clock sampler starts, then W warm-up semantics unchanged",
                      "l2": f"inputs larger than L2: {N_COPIES} rotating copies (~{N_COPIES * (B_er + B_tg) / 1e9:.2f} GB)"},
           "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
           "gpu": gpu_info(torch)}
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(prob)
    if extras:
        out["extras"] = extras
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def time_events(torch, fn, reps, spin_s=0.05):
    # untimed calls for spin_s first: the inputs were just generated on the host, and a GPU
    # that sat idle meanwhile runs its first launches below its clocks
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < spin_s:
        for _ in range(4):
            fn()
        torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run_extras(torch, pf, dev, peak):
    """Config 4 (K.v roofline, warm-started CG, Jacobi PCG §8(f) row f3), config 5 (64-part fused
    E+R) and the Newton warm start on a Neo-Hookean block (§8(f) row f1)."""
    from pfem_gen import config4, config5, warm_start
    ex = {}
    # ---------------- config 4: K.v fp64 + CG from zero / perturbed-exact warm start
    p4 = config4()
    E, N = p4.n_elems, p4.n_nodes
    t0 = time.perf_counter()
    m4 = pf.Mesh(torch.as_tensor(p4.coords, device=dev), torch.as_tensor(p4.conn, device=dev), dtype=torch.float64)
    torch.cuda.synchronize()
    prep = time.perf_counter() - t0
    mat4 = pf.Material("linear", "young_poisson", torch.as_tensor(p4.p0, device=dev), torch.as_tensor(p4.p1, device=dev))
    mask = torch.as_tensor(p4.mask, device=dev)
    f = torch.as_tensor(p4.f_ext, device=dev)
    vs = [torch.as_tensor(np.random.default_rng(i).standard_normal((1, N, 3)), device=dev) for i in range(3)]
    kv = torch.empty_like(vs[0])
    for i in range(5):
        pf.tangent_apply(m4, mat4, vs[i % 3], mask=mask, out=kv)
    torch.cuda.synchronize()
    it = [0]

    def kv_call():
        pf.tangent_apply(m4, mat4, vs[it[0] % 3], mask=mask, out=kv)
        it[0] += 1
    # a second mesh copy would double memory; config 4 arrays (~355 MB) exceed L2 on their own
    t_kv = time_events(torch, kv_call, 50)
    B_kv = bytes_tangent(E, N, 3, 1, 8, nh=False, mat_per_elem=1, masked=True)
    ex["config4_Kv"] = {"E": E, "us": t_kv * 1e3, "algorithmic_bytes": B_kv, "GBps": B_kv / (t_kv * 1e-3) / 1e9,
                        "frac": B_kv / (t_kv * 1e-3) / 1e9 / peak, "elements_per_s": E / (t_kv * 1e-3),
                        "prepare_s": prep}
    x0 = torch.zeros_like(f)
    pf.cg(m4, mat4, f, x0, mask=mask, tol=1e-8, max_iter=200)    # warm-up (graph build paths)
    torch.cuda.synchronize()

    def solve3(xs, **kw):
        # one timed solve per start, repeated 3 times, median time
        ts, out = [], None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = pf.cg(m4, mat4, f, xs, mask=mask, tol=1e-8, max_iter=20000, **kw)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return out[0], out[1], float(np.median(ts))

    def crossings(h):
        return {"iterations_to_1e-3": int(np.argmax(h < 1e-3)) if np.any(h < 1e-3) else None,
                "iterations_to_1e-6": int(np.argmax(h < 1e-6)) if np.any(h < 1e-6) else None}
    xz, rz, tz = solve3(x0, history=True)
    us, _ = pf.cg(m4, mat4, f, xz, mask=mask, tol=1e-12, max_iter=20000, history=False)
    xw = torch.as_tensor(warm_start(us.cpu().numpy(), p4.mask, seed=4004), device=dev)
    xw_out, rw, tw = solve3(xw, history=True)
    ex["config4_cg"] = {"tol": 1e-8, "timing": "median of 3 solves per start",
                        "zero": {"iterations": rz["iterations"], "time_to_tol_s": tz,
                                 "iterations_per_s": rz["iterations"] / tz,
                                 "ms_per_iteration": tz / max(1, rz["iterations"]) * 1e3,
                                 "true_rel_res": rz["true_rel_res_final"], **crossings(rz["history"])},
                        "warm": {"iterations": rw["iterations"], "time_to_tol_s": tw,
                                 "rel_res0": rw["rel_res0"], "true_rel_res": rw["true_rel_res_final"],
                                 **crossings(rw["history"])},
                        "speedup_iterations": rz["iterations"] / max(1, rw["iterations"]),
                        "speedup_time": tz / tw,
                        "warm_start": "u* (GPU CG to 1e-12) + 0.01 rms(u*) N(0,1) on free DOFs"}
    # §8(f) f3: Jacobi-preconditioned CG, same starts and tolerance
    pf.cg(m4, mat4, f, x0, mask=mask, tol=1e-8, max_iter=200, precond="jacobi")   # warm-up
    _, pz, tpz = solve3(x0, history=False, precond="jacobi")
    _, pw, tpw = solve3(xw, history=False, precond="jacobi")
    ex["config4_pcg_jacobi"] = {
        "tol": 1e-8,
        "zero": {"iterations": pz["iterations"], "time_to_tol_s": tpz, "ms_per_iteration": tpz / max(1, pz["iterations"]) * 1e3,
                 "true_rel_res": pz["true_rel_res_final"]},
        "warm": {"iterations": pw["iterations"], "time_to_tol_s": tpw, "true_rel_res": pw["true_rel_res_final"]},
        "iterations_vs_cg_zero": rz["iterations"] / max(1, pz["iterations"]),
        "iterations_vs_cg_warm": rw["iterations"] / max(1, pw["iterations"])}
    del m4, vs, kv
    torch.cuda.empty_cache()
    # ---------------- config 5: 64 ragged parts, NH fp32, fused E+R in one launch
    p5 = config5()
    E5, N5 = p5.n_elems, p5.n_nodes
    pe, pn = p5.parts()
    c5 = []
    for _ in range(N_COPIES):   # rotating copies (~0.4 GB): every call reads HBM, not L2 (§8(d4))
        m5 = pf.Mesh(torch.as_tensor(p5.coords, device=dev), torch.as_tensor(p5.conn, device=dev),
                     dtype=torch.float32, part_elem=pe, part_node=pn)
        mat5 = pf.Material("neohookean", "lame", torch.as_tensor(p5.p0, dtype=torch.float32, device=dev),
                           torch.as_tensor(p5.p1, dtype=torch.float32, device=dev))
        u5 = torch.as_tensor(p5.u, dtype=torch.float32, device=dev)
        outs = (torch.empty((1, 64), dtype=torch.float32, device=dev),
                torch.empty((1, E5), dtype=torch.float32, device=dev), torch.empty_like(u5))
        c5.append((m5, mat5, u5, outs))
    i5 = [0]

    def c5_call():
        m5_, mat5_, u5_, o5_ = c5[i5[0] % N_COPIES]
        pf.energy(m5_, mat5_, u5_, elem_energy=True, residual=True, out=o5_)
        i5[0] += 1
    for _ in range(6):
        c5_call()
    t5 = time_events(torch, c5_call, 60)
    B5 = bytes_energy_residual(E5, N5, 2, 1, 4, mat_per_elem=2, K=64)
    ex["config5_energy_residual"] = {"E": E5, "us": t5 * 1e3, "algorithmic_bytes": B5,
                                     "GBps": B5 / (t5 * 1e-3) / 1e9, "frac": B5 / (t5 * 1e-3) / 1e9 / peak,
                                     "elements_per_s": E5 / (t5 * 1e-3),
                                     "l2": f"{N_COPIES} rotating copies (inputs > L2)"}
    m5, mat5, u5, outs = c5[0]
    # §8(f) f2: the pretraining loss of the 64-sample batch through the hard-BC ansatz
    # u = phi (.) H, phi = distance to each plate's left edge / plate width (R28)
    phi5 = np.empty((N5, 2))
    for k in range(len(pn) - 1):
        x = p5.coords[pn[k]:pn[k + 1], 0]
        phi5[pn[k]:pn[k + 1]] = ((x - x.min()) / (x.max() - x.min()))[:, None]
    phi5t = torch.as_tensor(phi5, dtype=torch.float32, device=dev)
    f5 = torch.zeros_like(u5[0])
    pl_out = (torch.empty((), dtype=torch.float64, device=dev), torch.empty((1, 64), dtype=torch.float32, device=dev),
              torch.empty_like(u5), torch.empty_like(u5))
    for _ in range(5):
        pf.pretrain_loss(m5, mat5, u5, phi=phi5t, f_ext=f5, out=pl_out)
    tpl = time_events(torch, lambda: pf.pretrain_loss(m5, mat5, u5, phi=phi5t, f_ext=f5, out=pl_out), 50)
    ex["config5_pretrain_loss"] = {"us": tpl * 1e3, "samples": 64, "samples_per_s": 64 / (tpl * 1e-3),
                                   "loss": float(pl_out[0]),
                                   "launches": "ansatz + fused energy/residual with the gradient epilogue in its writes and the loss in kernel B's last CTA",
                                   "note": "timed back-to-back on one copy (partly L2-resident)"}
    del m5, outs, c5
    torch.cuda.empty_cache()
    # ---------------- configs 1 and 2 (BASELINE configs[0], configs[1]): latency of the tiny
    # case; config 2 fused E+R over 32 fields in fp32 and fp64 (3 rotating copies > L2)
    from pfem_gen import config1, config2
    p1 = config1()
    m1 = pf.Mesh(torch.as_tensor(p1.coords, device=dev), torch.as_tensor(p1.conn, device=dev), dtype=torch.float64)
    mat1 = pf.Material("linear", "young_poisson", torch.as_tensor(p1.p0, device=dev), torch.as_tensor(p1.p1, device=dev))
    u1 = torch.as_tensor(p1.u, device=dev)
    out1 = (torch.empty((1, 1), dtype=torch.float64, device=dev), torch.empty((1, p1.n_elems), dtype=torch.float64, device=dev),
            torch.empty_like(u1))
    for _ in range(5):
        pf.energy(m1, mat1, u1, elem_energy=True, residual=True, out=out1)
    t1 = time_events(torch, lambda: pf.energy(m1, mat1, u1, elem_energy=True, residual=True, out=out1), 200)
    ex["config1_energy_residual"] = {"E": p1.n_elems, "us": t1 * 1e3, "note": "latency: one E+R call on 450 T3 (fp64)"}
    for dt_name, tdt, sz in (("f32", torch.float32, 4), ("f64", torch.float64, 8)):
        p2 = config2(dtype=dt_name)
        E2, N2, S2 = p2.n_elems, p2.n_nodes, p2.u.shape[0]
        cps = []
        for c in range(3):
            m2 = pf.Mesh(torch.as_tensor(p2.coords, device=dev), torch.as_tensor(p2.conn, device=dev), dtype=tdt)
            mat2 = pf.Material("linear", "young_poisson", torch.as_tensor(p2.p0, dtype=tdt, device=dev),
                               torch.as_tensor(p2.p1, dtype=tdt, device=dev))
            u2 = torch.as_tensor(p2.u, dtype=tdt, device=dev)
            cps.append((m2, mat2, u2, (torch.empty((S2, 1), dtype=tdt, device=dev),
                                       torch.empty((S2, E2), dtype=tdt, device=dev), torch.empty_like(u2))))
        for i in range(6):
            m2, mat2, u2, o2 = cps[i % 3]
            pf.energy(m2, mat2, u2, elem_energy=True, residual=True, out=o2)
        i2 = [0]

        def c2_call():
            m2, mat2, u2, o2 = cps[i2[0] % 3]
            pf.energy(m2, mat2, u2, elem_energy=True, residual=True, out=o2)
            i2[0] += 1
        t2 = time_events(torch, c2_call, 60)
        B2 = bytes_energy_residual(E2, N2, 2, S2, sz, True, 1)
        ex[f"config2_energy_residual_{dt_name}"] = {"E": E2, "S": S2, "us": t2 * 1e3, "algorithmic_bytes": B2,
                                                    "GBps": B2 / (t2 * 1e-3) / 1e9, "frac": B2 / (t2 * 1e-3) / 1e9 / peak,
                                                    "element_samples_per_s": E2 * S2 / (t2 * 1e-3),
                                                    "l2": "3 rotating copies"}
        del cps
    torch.cuda.empty_cache()
    # ---------------- §8(f) f4: steady heat conduction on the config-3 mesh (4 fields, fp32)
    from pfem_gen import config3
    p3 = config3()
    E3, N3 = p3.n_elems, p3.n_nodes
    m3 = pf.Mesh(torch.as_tensor(p3.coords, device=dev), torch.as_tensor(p3.conn, device=dev), dtype=torch.float32)
    rng = np.random.default_rng(3009)
    k3 = torch.as_tensor(np.exp(0.5 * rng.standard_normal(E3)), dtype=torch.float32, device=dev)
    T3s = [torch.as_tensor(rng.standard_normal((4, N3)), dtype=torch.float32, device=dev) for _ in range(3)]
    f3 = torch.as_tensor(0.01 * rng.standard_normal(N3), dtype=torch.float32, device=dev)
    for i in range(3):
        pf.heat(m3, k3, T3s[i], f=f3)
    ih = [0]

    def heat_call():
        pf.heat(m3, k3, T3s[ih[0] % 3], f=f3)
        ih[0] += 1
    th = time_events(torch, heat_call, 30)
    B_h = E3 * (16 + 9 * 4 + 4 + 4) + 4 * (N3 * 4 * 2 + E3 * 4 + 4) + N3 * 4
    ih[0] = 0

    def heat_otf_call():
        pf.heat(m3, k3, T3s[ih[0] % 3], f=f3, geometry_on_the_fly=True)
        ih[0] += 1
    heat_otf_call()
    th_otf = time_events(torch, heat_otf_call, 30)
    ex["heat_config3_mesh"] = {"E": E3, "S": 4, "us": th * 1e3, "us_geometry_on_the_fly": th_otf * 1e3,
                               "algorithmic_bytes": B_h,
                               "GBps": B_h / (th * 1e-3) / 1e9, "frac": B_h / (th * 1e-3) / 1e9 / peak,
                               "element_samples_per_s": E3 * 4 / (th * 1e-3),
                               "kernels": "k_heat_elem + k_heat_totals + k_heat_flux (CSR gather, element gradient re-formed per entry)"}
    del m3, T3s
    torch.cuda.empty_cache()
    # ---------------- §8(f) f1: Newton-Raphson warm start on a Neo-Hookean block (fp64)
    from pfem_gen import newton_block
    pn_ = newton_block(33, traction=(0.05, 0.0, 0.02))
    mn = pf.Mesh(torch.as_tensor(pn_.coords, device=dev), torch.as_tensor(pn_.conn, device=dev), dtype=torch.float64)
    matn = pf.Material("neohookean", "lame", torch.as_tensor(pn_.p0, device=dev), torch.as_tensor(pn_.p1, device=dev))
    fn = torch.as_tensor(pn_.f_ext, device=dev)
    maskn = torch.as_tensor(pn_.mask, device=dev)
    un0 = torch.zeros_like(fn)
    tol_n = 1e-9 * float(np.linalg.norm(pn_.f_ext))
    pf.newton(mn, matn, un0, f_ext=fn, mask=maskn, tol=tol_n, max_newton=1, cg_tol=1e-3)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    uz, nz = pf.newton(mn, matn, un0, f_ext=fn, mask=maskn, tol=tol_n, cg_tol=1e-10)
    tnz = time.perf_counter() - t0
    uw0 = torch.as_tensor(warm_start(uz.cpu().numpy(), pn_.mask, seed=6004), device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, nw = pf.newton(mn, matn, uw0, f_ext=fn, mask=maskn, tol=tol_n, cg_tol=1e-10)
    tnw = time.perf_counter() - t0
    ex["newton_nh_block"] = {
        "mesh": f"unit cube 33^3 nodes, Kuhn T4 ({pn_.n_elems} tets), NH mu=0.4 lam=0.6, clamped z=0, "
                "top traction (0.05, 0, 0.02)", "tol_abs": tol_n, "cg_tol": 1e-10,
        "zero": {"newton_iterations": nz["iterations"], "cg_iterations": nz["cg_iterations"], "time_s": tnz,
                 "history": [float(x) for x in nz["history"]]},
        "warm": {"newton_iterations": nw["iterations"], "cg_iterations": nw["cg_iterations"], "time_s": tnw,
                 "history": [float(x) for x in nw["history"]]},
        "warm_start": "U* (converged Newton) + 0.01 rms(U*) N(0,1) on free DOFs"}
    # ---------------- §8(f) f4: the paper's quadrilateral Newton rows (Table 1 beam / Cook,
    # P:474-480): zero start vs perturbed-exact warm start, fp64
    from pfem_gen import beam_q4, cook_q8, smooth_warm_start
    for name, mk, paper in (("newton_beam_q4", beam_q4, "4.90 -> 1.34 Newton iterations (P:474)"),
                            ("newton_cook_q8", cook_q8, "8.38 -> 1.55 Newton iterations (P:480)")):
        pq = mk()
        mq = pf.Mesh(torch.as_tensor(pq.coords, device=dev), torch.as_tensor(pq.conn, device=dev),
                     dtype=torch.float64, elem_type=pq.elem)
        matq = pf.Material(pq.model, pq.param_kind, torch.as_tensor(pq.p0, device=dev),
                           torch.as_tensor(pq.p1, device=dev))
        fq = torch.as_tensor(pq.f_ext, device=dev)
        maskq = torch.as_tensor(pq.mask, device=dev)
        tol_q = 1e-10 * float(np.linalg.norm(pq.f_ext))
        uq0 = torch.zeros_like(fq)
        pf.newton(mq, matq, uq0, f_ext=fq, mask=maskq, tol=tol_q, max_newton=1, cg_tol=1e-3)   # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        uz, rz_ = pf.newton(mq, matq, uq0, f_ext=fq, mask=maskq, tol=tol_q, cg_tol=1e-10)
        tz_ = time.perf_counter() - t0
        uw0 = torch.as_tensor(smooth_warm_start(uz.cpu().numpy(), pq.coords, pq.mask, seed=8004), device=dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rw_ = pf.newton(mq, matq, uw0, f_ext=fq, mask=maskq, tol=tol_q, cg_tol=1e-10)
        tw_ = time.perf_counter() - t0
        ex[name] = {"mesh": f"{pq.n_elems} {pq.elem.upper()} elements, {pq.n_nodes} nodes", "tol_abs": tol_q,
                    "zero": {"newton_iterations": rz_["iterations"], "cg_iterations": rz_["cg_iterations"],
                             "converged": rz_["converged"], "time_s": tz_},
                    "warm": {"newton_iterations": rw_["iterations"], "cg_iterations": rw_["cg_iterations"],
                             "converged": rw_["converged"], "time_s": tw_},
                    "warm_start": "U* + 0.01 rms(U*) Phi(X)/rms(Phi), Phi a smooth seeded Fourier field (free DOFs)",
                    "paper_context": paper + " (GRF test cases, Transolver warm start; other hardware)"}
    return ex


# ----------------------------------------------------------------------------- CPU oracle
def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(prob, min_s=10.0, min_s1=5.0):
    """The oracle as it stands (fp64, OpenMP on all host cores) on the bench step itself: the
    4 fields of config 3 on the full mesh, energy + residual + tangent, repeated until at least
    `min_s` seconds of CPU work (about 10-30 s, a bounded sample); beside it the same oracle on
    one thread (a leading sub-mesh of 200k tets, 1 field, at least `min_s1` seconds) and the
    oracle CG on config 4."""
    from oracle import oracle
    om = oracle.prepare_problem(prob)
    u = prob.u
    v = np.random.default_rng(3005).standard_normal(u.shape)

    def timed(mesh, uu, vv, floor):
        reps, t0 = 0, time.perf_counter()
        while True:
            mesh.energy(uu)
            mesh.residual(uu)
            mesh.tangent(vv, u=uu)
            reps += 1
            dt = time.perf_counter() - t0
            if dt >= floor:
                return reps, dt
    reps, dt = timed(om, u, v, min_s)
    sub = submesh(prob, 200_000)
    oms = oracle.prepare_problem(sub)
    oracle.set_threads(1)
    reps1, dt1 = timed(oms, u[:1], v[:1], min_s1)
    oracle.set_threads(0)
    cg = cpu_cg_config4(oracle)
    return {"value": prob.n_elems * prob.n_samples * reps / dt, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
            "cg_config4": cg,
            "sample": f"the config-3 step ({prob.n_samples} fields, full mesh, {prob.n_elems} tets): energy + residual + "
                      f"tangent, fp64, {reps} repetitions in {dt:.1f} s",
            "single_thread": {"value": sub.n_elems * reps1 / dt1, "unit": UNIT, "cores": 1,
                              "sample": f"leading {sub.n_elems} tets of config 3, 1 field, {reps1} repetitions in {dt1:.1f} s"},
            "cpu_model": cpu_model()}


def cpu_cg_config4(oracle, n_timed=20):
    """The oracle CG on config 4: 20 iterations timed on all host cores, the
    time to tolerance extrapolated with the oracle's own iteration counts to 1e-8 (zero and
    warm start, tests/golden/config4_cg.json, written by an oracle-only script)."""
    from pfem_gen import config4
    p4 = config4()
    om = oracle.prepare_problem(p4)
    t0 = time.perf_counter()
    _, rep = om.cg(p4.f_ext, p4.mask, np.zeros_like(p4.f_ext), tol=1e-30, max_iter=n_timed, history=False)
    dt = time.perf_counter() - t0
    per_it = dt / (n_timed + 3)   # + r0, the lifted rhs and the final true-residual products
    out = {"timed_iterations": n_timed, "seconds": dt, "seconds_per_iteration": per_it, "cores": cpu_cores(),
           "method": "extrapolated from 20 timed iterations x the oracle's iteration count"}
    gp = os.path.join(ROOT, "tests", "golden", "config4_cg.json")
    if os.path.exists(gp):
        with open(gp) as fh:
            g = json.load(fh)
        for start in ("zero", "warm"):
            k = g[start]["runs"]["0"]["iterations"]
            out[start] = {"iterations": k, "time_to_tol_s": k * per_it}
    return out


def gpu_info(torch):
    info = {"name": torch.cuda.get_device_name(), "sms": torch.cuda.get_device_properties(0).multi_processor_count}
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=driver_version", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=10).stdout.strip().splitlines()
        info["driver"] = out[0] if out else None
    except Exception:
        info["driver"] = None
    return info


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def submesh(prob, n_elems):
    """First n_elems elements of a problem (a valid mesh: unused nodes carry no stiffness)."""
    from pfem_gen.configs import Problem
    return Problem(prob.name + f"[:{n_elems}]", prob.dim, prob.coords, prob.conn[:n_elems], prob.model,
                   prob.param_kind, prob.p0 if len(prob.p0) == 1 else prob.p0[:n_elems],
                   prob.p1 if len(prob.p1) == 1 else prob.p1[:n_elems], prob.u, prob.dtype)


def run_reference(args, budget_s=150.0):
    """The reference arm of this tier: the CPU oracle as it stands, timed on this box's host
    cores on the same workload / metric; each step is the config-3 step (all fields) on a leading
    sub-mesh sized so that the W + K steps fit in ~budget_s (the full mesh when they do)."""
    world, rank, _ = dist_info()
    if rank != 0:
        return
    from pfem_gen import config3
    from oracle import oracle
    prob = config3()
    probe = submesh(prob, 100_000)
    om = oracle.prepare_problem(probe)
    u = prob.u
    v = np.random.default_rng(3005).standard_normal(u.shape)
    t0 = time.perf_counter()
    om.energy(u); om.residual(u); om.tangent(v, u=u)
    per_elem = (time.perf_counter() - t0) / probe.n_elems
    n_el = int(min(prob.n_elems, max(10_000, budget_s / max(1, args.steps + args.warmup) / per_elem)))
    sub = submesh(prob, n_el)
    om = oracle.prepare_problem(sub)

    def one():
        om.energy(u)
        om.residual(u)
        om.tangent(v, u=u)

    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt = (time.perf_counter() - t0) / args.steps
    value = n_el * prob.n_samples / dt
    sample = (f"config 3, all {prob.n_samples} fields per step, leading {n_el} of {prob.n_elems} tets: "
              "oracle energy + residual + tangent (fp64, OpenMP)")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, pfem_gen)", "impl": "reference",
           "config": {"workload": "config3", "n_elems": prob.n_elems, "n_nodes": prob.n_nodes, "sample": sample},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without a launcher: start N ranks ourselves (one process per GPU, torchrun,
        # rendezvous on 127.0.0.1) and return rank 0's exit status
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
        return
    run_gpu(args)


if __name__ == "__main__":
    main()
