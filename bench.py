#!/usr/bin/env python
"""Benchmark of the B200-native reduced-objective hot path (BASELINE.json metric:
"E+grad evals/sec and ms/timestep (L-BFGS, eps=1e-5); % of HBM roofline").

Headline workload (N=1 default): BASELINE.json configs[2] = config 3, the largest
single-GPU configuration (32x32x128 jittered Kuhn bar, 786,432 tets, per-tet E,
d=32, 5x256 ELU decoder, seed 2), fp32 storage / fp64 arithmetic, the
timestep-0 objective E(z) = |f(z) - qbar|_M^2/(2h^2) + P(f(z)).  One bench
"step" = one E+grad evaluation at a fresh seeded z ~ N(0, 0.5^2 I), inputs
resident in HBM; L2 is flushed before every timed step (a 512 MiB write; W_out
alone is 418 MB, larger than L2).  ms/timestep over all 100 configured
timesteps (5 m/s impulse at t=0) is reported with iteration counts and the
exit-code histogram (diagnostics.cpp:153-172 layout).

Per-config records ("records") carry the other BASELINE configs, each with its
own roofline fraction and CPU baseline:
  c1  fp64, 100 timesteps + E+grad evals/s
  c2  fp64, 200 timesteps + E+grad evals/s (+ value-only evals/s); c2f the same in fp32 storage
  c4  4096 z on the c2 problem (tcgen05 GEMMs), evals/s + tensor fraction
  c5  1024 latent pairs on the c2 problem, order-2 Lipschitz loss, ms

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c1|c2|c2f|c3] [--records c1,c2,c4,c5|none]

Multi-GPU: single-instance solves (c1-c3) do not shard: every rank
runs an independent replica, value = evals of all ranks / max-over-ranks time.
c4 shards the latent batch and c5 the pairs across ranks (no data-path
collective; timing is max over ranks).  --gpus N without a torchrun environment
re-launches itself under torch.distributed.run with N ranks.
--impl reference times the reference's CPU algorithm (the oracle port: the
reference itself cannot be built here) on all host cores, rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLUSH_BYTES = 512 << 20
# dram__bytes_read.sum + dram__bytes_write.sum per launch of the reported kernel, from the
# committed ncu --set full captures (profiles/); None until captured for that path.
TRAFFIC = {
    # profiles/r01_solve_c2_v5_full.txt: one c2 fp64 E+grad eval (ncu flushes caches before the
    # launch, like the bench's L2 flush): dram read 75.42 MB + write 5.79 MB
    ("c2", True): 81.20e6,
    # profiles/r02_launches_c3.txt: one c3 evaluation's streaming kernels under ncu (caches flushed
    # before every kernel, so the CSR forces the gather re-reads come from DRAM here, from L2 in the
    # bench): out_fwd 438.8 + 1.2, elem 67.4 + 6.9, vjp_gather 475.1 + 0.3 MB (launches 3-5)
    ("c3", False): 989.7e6,
}
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
LATENT = {"c1": 8, "c2": 16, "c2f": 16, "c3": 32}


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def algorithmic_bytes(n, h, E, w, per_tet_material=False, want_grad=True):
    """Per-eval bytes: E+grad w(2nh + 9n) + E(16 + 10w) [+ 2wE];
    value-only w(nh + 8n) + E(16 + 10w) [+ 2wE]."""
    mat = 2 * w * E if per_tet_material else 0
    if want_grad:
        return w * (2 * n * h + 9 * n) + E * (16 + 10 * w) + mat
    return w * (n * h + 8 * n) + E * (16 + 10 * w) + mat


class ClockSampler:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[1]) for s in self.samples if len(s) > 8 and s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if len(s) > 8 and s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) > 8:
                for nm, v in zip(names, s[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def maybe_relaunch(argv, gpus):
    """--gpus N outside torchrun: re-launch under torch.distributed.run with N ranks."""
    if gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + argv
    sys.exit(subprocess.call(cmd))


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        return ws, rank, local, dist
    return 1, 0, local, None


class Ranks:
    """max / sum over ranks (NCCL on the rank's GPU); identity at world size 1."""

    def __init__(self, ws, rank, local, dist):
        self.ws, self.rank, self.local, self.dist = ws, rank, local, dist

    def _red(self, v, op):
        if not self.dist:
            return float(v)
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64, device=f"cuda:{self.local}")
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v):
        return self._red(v, self.dist.ReduceOp.MAX if self.dist else None)

    def sum(self, v):
        return self._red(v, self.dist.ReduceOp.SUM if self.dist else None)

    def barrier(self):
        if self.dist:
            self.dist.barrier()


# ------------------------------------------------------------------------------------ CPU side
def timestep0_qbar_oracle(ob):
    from paper_2409_03807_b200 import configs
    X = ob.mesh_arrays()[0]
    free = np.nonzero(ob.mesh_arrays()[4] >= 0)[0]
    return X[free].reshape(-1) + configs.DT ** 2 * np.tile(configs.GRAVITY, free.size)


_ORACLES = {}


def oracle_problem(name):
    from oracle import pyoracle
    key = "c2" if name in ("c2f", "c4", "c5") else name
    if key not in _ORACLES:
        _ORACLES[key] = pyoracle.problem(key)
    return _ORACLES[key]


def cpu_eval_rate(name, evals, threads, rng_seed=11, want_grad=True):
    """Oracle (C++ restatement of the reference, -O3) evals/s on `threads` host threads."""
    from paper_2409_03807_b200 import configs
    ob = oracle_problem(name)
    qbar = timestep0_qbar_oracle(ob)
    Z = 0.5 * np.random.default_rng(rng_seed).standard_normal((evals, LATENT.get(name, 16)))
    t0 = time.perf_counter()
    ob.eval_batch(Z, qbar=qbar, dt=configs.DT, threads=threads, want_grad=want_grad)
    dt = time.perf_counter() - t0
    return evals / dt, dt


def cpu_baseline_eval(name, sample):
    rate, dt = cpu_eval_rate(name, sample, 1)
    return {"value": rate, "unit": "evals/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
            "sample": f"{sample} E+grad evals of {name} on 1 host core (oracle C++ -O3, {dt:.1f} s); "
                      "the reference is single-threaded"}


def cpu_baseline_steps(name, steps):
    """Oracle reduced_step loop (reference reduced_step + lbfgs_minimize) on 1 core."""
    from paper_2409_03807_b200 import configs
    ob = oracle_problem(name)
    t0 = time.perf_counter()
    res = ob.simulate(steps, configs.solver_config(), gravity=configs.GRAVITY)
    dt = time.perf_counter() - t0
    return {"ms_per_timestep": 1e3 * dt / steps, "timesteps": steps, "cores": 1, "kind": "port",
            "mean_iterations": float(np.mean(res["iterations"])),
            "exit_histogram": {str(int(c)): int((res["codes"] == c).sum()) for c in np.unique(res["codes"])}}


# ------------------------------------------------------------------------------------ GPU side
def lib_and_P():
    import paper_2409_03807_b200 as P
    return P, P.lib()


def bench_evals(P, L, sysm, Z, want_grad=True):
    k = Z.shape[0]
    ev, of, Es = np.zeros(k), np.zeros(k), np.zeros(k)
    P.check(L.lsb_bench_evals_ex(sysm.handle, k, P.dptr(np.ascontiguousarray(Z)), FLUSH_BYTES, int(want_grad),
                                 P.dptr(ev), P.dptr(of), P.dptr(Es)))
    return ev, of, Es


def run_timesteps(P, L, pr, sysm, T):
    import ctypes as C
    from paper_2409_03807_b200 import configs
    st = pr.initial_state()
    sysm.set_state(st)
    sysm.set_external_force(P.gravity_force(pr.mesh, sysm.mass, configs.GRAVITY))
    cfg = configs.solver_config()
    step_ms = np.zeros(T)
    reps = (P._capi.lsb_exit_report * T)()
    c = cfg._c()
    P.check(L.lsb_bench_steps(sysm.handle, T, C.byref(c), 0, FLUSH_BYTES, P.dptr(step_ms), reps))
    iters = np.array([reps[i].iterations for i in range(T)])
    vevals = np.array([reps[i].value_evals for i in range(T)])
    gevals = np.array([reps[i].grad_evals for i in range(T)])
    codes = np.array([reps[i].code for i in range(T)])
    return {
        "timesteps": T, "ms_per_timestep": float(step_ms.mean()), "ms_total": float(step_ms.sum()),
        "mean_iterations": float(iters.mean()), "max_iterations": int(iters.max()),
        "exit_histogram": {str(int(k)): int((codes == k).sum()) for k in np.unique(codes)},
        "evals_per_timestep": float((vevals).mean()), "grad_evals_per_timestep": float(gevals.mean()),
        "iterations": iters.tolist(),
        "timed": "each step bracketed by CUDA events on the context stream, L2 flushed before each",
    }


def single_instance(name, K, W, T, R, want_cpu, cpu_sample, e2e=True):
    """E+grad evals/s (device-timed), value-only evals/s, ms/timestep over T steps,
    roofline of the evaluation, e2e through the C ABI."""
    import ctypes as C
    P, L = lib_and_P()
    from paper_2409_03807_b200 import configs
    pr = configs.build(name)
    sysm = pr.system(device=R.local)
    spec = pr.spec
    n, r, h, E = pr.model.n, pr.model.r, spec.width, pr.mesh.num_elements()
    w = 8 if sysm.precision == "fp64" else 4
    qbar = configs.timestep0_qbar(pr, sysm.mass)
    sysm.set_inertia(qbar, configs.DT)
    Z = configs.gaussian_latents(100 + R.rank, K + W, r)
    bench_evals(P, L, sysm, Z[:W])  # warm-up (untimed)
    R.barrier()
    launches0 = sysm.launch_count()
    ev_ms, of_ms, Es = bench_evals(P, L, sysm, Z[W:])
    launches = sysm.launch_count() - launches0
    t_ms = R.max(float(ev_ms.sum()))
    value = R.ws * K / (t_ms * 1e-3)
    # value-only evaluations (lsb_eval with grad == NULL)
    bench_evals(P, L, sysm, Z[:W], want_grad=False)
    vo_ms, _, _ = bench_evals(P, L, sysm, Z[W:], want_grad=False)
    vo_t = R.max(float(vo_ms.sum()))
    value_only = R.ws * K / (vo_t * 1e-3)
    # the same evaluations after a write flush FOLLOWED by a read pass over a second buffer: the write
    # flush leaves L2 full of dirty lines whose write-back otherwise lands inside the timed evaluation
    # (reported beside the headline, which keeps the plain write flush)
    os.environ["LSB_FLUSH_MODE"] = "readback"
    try:
        bench_evals(P, L, sysm, Z[:W])
        cl_ms, _, _ = bench_evals(P, L, sysm, Z[W:])
    finally:
        os.environ.pop("LSB_FLUSH_MODE", None)
    cl_t = R.max(float(cl_ms.sum()))
    steps = run_timesteps(P, L, pr, sysm, T)
    steps["ms_per_timestep"] = R.max(steps["ms_per_timestep"])
    # e2e: the reference-facing C-ABI call lsb_eval (host z in, host E and grad out, the copies
    # inside every call), K back-to-back calls timed on the host clock
    sysm.set_inertia(qbar, configs.DT)
    Ze = np.ascontiguousarray(configs.gaussian_latents(7, K + W, r))
    Ee, Ge = np.zeros(K + W), np.zeros((K + W, r))
    secs = C.c_double()
    P.check(L.lsb_bench_e2e(sysm.handle, W, P.dptr(Ze[:W]), P.dptr(Ee[:W]), P.dptr(Ge[:W]), C.byref(secs)))
    P.check(L.lsb_bench_e2e(sysm.handle, K, P.dptr(np.ascontiguousarray(Ze[W:])), P.dptr(Ee[W:]),
                            P.dptr(Ge[W:]), C.byref(secs)))
    e2e_t = R.max(secs.value)
    py_t = 0.0
    for k in range(W, W + K):
        t0 = time.perf_counter()
        sysm.eval(Ze[k])
        py_t += time.perf_counter() - t0
    py_t = R.max(py_t)
    hbm, _, peak_kind = peaks()
    per_tet = spec.young[1] > spec.young[0]
    alg = algorithmic_bytes(n, h, E, w, per_tet)
    alg_vo = algorithmic_bytes(n, h, E, w, per_tet, want_grad=False)
    solve = sysm.solve_kernel_info()
    dur_s = float(ev_ms.mean()) * 1e-3
    achieved = alg / dur_s / 1e9
    if solve["in_use"]:
        kname = "solve_kernel (persistent cooperative cluster kernel, one launch per evaluation)"
    else:
        kname = ("multi-kernel evaluation (ctrl_fast -> out_fwd_tma -> elem -> vjp_gather_tma -> ctrl_fast, "
                 "one CUDA graph per evaluation)")
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "frac_of_nominal_8TBs": achieved / 8000.0,
            "traffic": TRAFFIC.get((name, solve["in_use"])), "kernel": kname, "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": alg,
            "algorithmic_formula": "w(2nh+9n)+E(16+10w)[+2wE] per E+grad eval (SURVEY 8d)",
            "value_only_frac": alg_vo / (float(vo_ms.mean()) * 1e-3) / 1e9 / hbm}
    clean = {"value": R.ws * K / (cl_t * 1e-3), "unit": "evals/s", "ms_per_eval": cl_t / K,
             "roofline_frac": alg / (float(cl_ms.mean()) * 1e-3) / 1e9 / hbm,
             "l2": f"{FLUSH_BYTES >> 20} MiB write flush, then a {FLUSH_BYTES >> 20} MiB read pass over a second buffer "
                   "(outside the timed interval): L2 holds none of the inputs and no dirty lines of the flush"}
    rec = {
        "config": {"workload": f"{name}: {spec.grid[0]}x{spec.grid[1]}x{spec.grid[2]} Kuhn bar, {E} tets, n={n}, "
                               f"d={r}, {spec.hidden_layers}x{h} ELU, {sysm.precision}"
                               + (", jitter 0.1 cell, per-tet E in [5e4, 5e5], 5 m/s impulse" if per_tet else "")
                               + "; one E+grad eval per step (timestep-0 objective)",
                   "l2": f"flushed before every timed step ({FLUSH_BYTES >> 20} MiB write)",
                   "parallelism": f"replicas x{R.ws}"},
        "metric": "E+grad evals/sec", "value": value, "unit": "evals/s", "ms_per_eval": t_ms / K, "evals": K,
        "value_only_evals_per_s": value_only, "clean_l2": clean,
        "dtype": "f64" if w == 8 else "f32 storage / f64 arithmetic",
        "timesteps": steps, "roofline": roof,
        "e2e": {"value": R.ws * K / e2e_t if e2e_t > 0 else None, "unit": "evals/s", "h2d_bytes_per_step": 8 * r,
                "d2h_bytes_per_step": 8 * (1 + r), "api": "lsb_eval (C ABI), host buffers",
                "l2": "back-to-back calls, no flush (as inside a solve)",
                "python_binding_value": R.ws * K / py_t if py_t > 0 else None},
        "gpu_launches": int(launches), "energy_check": float(Es[0]),
        "dev_flags": sysm.dev_flags() or None, "solve_path": solve["reason"],
    }
    if want_cpu and R.rank == 0 and R.ws == 1:
        cb = cpu_baseline_eval(name, cpu_sample)
        if name == "c1":
            cb["timesteps"] = cpu_baseline_steps("c1", T)
        elif name in ("c2", "c2f"):
            cb["timesteps"] = cpu_baseline_steps(name, 3)
            cb["timesteps"]["note"] = "first 3 timesteps only (CPU budget)"
        else:
            cb["timesteps"] = {"ms_per_timestep_extrapolated": 1e3 / cb["value"] * steps["evals_per_timestep"],
                               "note": "extrapolated: CPU ms per E+grad eval x the GPU run's mean evaluations "
                                       "per timestep (a CPU c3 timestep takes tens of seconds)"}
        rec["cpu_baseline"] = cb
    sysm.close()
    return rec


def batched_record(K, W, R, want_cpu):
    """c4: E+grad for 4096 z on the c2 problem (fp32 batched path, tcgen05 GEMMs)."""
    P, L = lib_and_P()
    from paper_2409_03807_b200 import configs
    from paper_2409_03807_b200 import replicas
    pr = configs.build("c2")
    sysm = pr.system("fp32", device=R.local)
    n, r, h = pr.model.n, pr.model.r, pr.spec.width
    sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
    Bt = 4096
    Z = configs.latent_batch_c4(r, Bt)
    lo, hi = replicas.shard_range(Bt, R.ws, R.rank)
    Zl = np.ascontiguousarray(Z[lo:hi])
    B = hi - lo
    E, G = np.zeros(B), np.zeros((B, r))
    ms = np.zeros(max(W, 1))
    P.check(L.lsb_bench_batched(sysm.handle, 0, B, P.dptr(Zl), None, max(W, 1), FLUSH_BYTES, P.dptr(ms),
                                P.dptr(E), P.dptr(G), None))
    reps = max(1, min(K, 10))
    ms = np.zeros(reps)
    R.barrier()
    l0 = sysm.launch_count()
    P.check(L.lsb_bench_batched(sysm.handle, 0, B, P.dptr(Zl), None, reps, FLUSH_BYTES, P.dptr(ms),
                                P.dptr(E), P.dptr(G), None))
    launches = sysm.launch_count() - l0
    t = R.max(float(ms.mean()))
    t0 = time.perf_counter()
    E2, G2 = sysm.eval_batched(Zl)
    e2e_t = R.max(time.perf_counter() - t0)
    hbm, bf16, peak_kind = peaks()
    gemm_flops = 2 * (2.0 * n * h * Bt)  # output GEMM + VJP GEMM (fp32-equivalent)
    achieved = gemm_flops / (t * 1e-3) / 1e12
    rec = {
        "config": {"workload": f"c4: {Bt} z ~ N(0, 0.25 I) (substream(3,0)) on the c2 problem, timestep-0 objective, "
                               "fp32 arithmetic with fp64 reductions; output and VJP GEMMs on tcgen05 (3xTF32)",
                   "l2": f"flushed before every call ({FLUSH_BYTES >> 20} MiB write)",
                   "parallelism": f"batch sharded x{R.ws}"},
        "metric": "E+grad evals/sec", "value": Bt / (t * 1e-3), "unit": "evals/s", "ms_per_batch": t, "reps": reps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": bf16, "unit": "TFLOP/s",
                     "frac": achieved / bf16, "traffic": None,
                     "algorithmic_flops_per_batch": gemm_flops, "peak_kind": peak_kind + ", dense bf16",
                     "note": "GEMM flops (2 x 2nhB) over the whole batch time; 3xTF32 issues 3 MMA passes per "
                             "product; the unfused HBM floor is ~0.54 ms (SURVEY 8d)",
                     "hbm_floor_frac": 0.54 / t},
        "e2e": {"value": Bt / e2e_t, "unit": "evals/s", "h2d_bytes_per_step": 8 * B * r,
                "d2h_bytes_per_step": 8 * B * (1 + r), "api": "lsb_eval_batched (C ABI), host buffers"},
        "gpu_launches": int(launches // reps), "energy_check": float(E[0]) if B else None,
        "timed": "CUDA events on the context stream around each lsb_eval_batched call (includes its Z upload and "
                 "E/G download, ~1 MB)",
    }
    if want_cpu and R.rank == 0 and R.ws == 1:
        sample = 64
        rate, dt = cpu_eval_rate("c4", sample, 1)
        ncores = os.cpu_count() or 1
        rate_all, dt_all = cpu_eval_rate("c4", 4 * ncores, ncores)
        rec["cpu_baseline"] = {"value": rate, "unit": "evals/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
                               "sample": f"{sample} E+grad evals of the c2 objective on 1 core ({dt:.1f} s)",
                               "all_cores": {"value": rate_all, "cores": ncores,
                                             "sample": f"{4 * ncores} evals, std::thread over z ({dt_all:.1f} s)"}}
    sysm.close()
    return rec


def lipschitz_record(K, W, R, want_cpu):
    """c5: order-2 Lipschitz loss over 1024 pairs on the c2 problem (elastic potential)."""
    P, L = lib_and_P()
    from paper_2409_03807_b200 import configs
    from paper_2409_03807_b200 import replicas
    pr = configs.build("c2")
    sysm = pr.system("fp32", device=R.local)
    r = pr.model.r
    Pt = 1024
    Z1, Z2 = configs.latent_pairs_c5(r, Pt)
    lo, hi = replicas.shard_range(Pt, R.ws, R.rank)
    Z1l, Z2l = np.ascontiguousarray(Z1[lo:hi]), np.ascontiguousarray(Z2[lo:hi])
    loss = np.zeros(1)
    ms = np.zeros(1)
    P.check(L.lsb_bench_batched(sysm.handle, 1, hi - lo, P.dptr(Z1l), P.dptr(Z2l), 1, FLUSH_BYTES, P.dptr(ms),
                                None, None, P.dptr(loss)))
    reps = max(1, min(K, 3))
    ms = np.zeros(reps)
    R.barrier()
    l0 = sysm.launch_count()
    P.check(L.lsb_bench_batched(sysm.handle, 1, hi - lo, P.dptr(Z1l), P.dptr(Z2l), reps, FLUSH_BYTES, P.dptr(ms),
                                None, None, P.dptr(loss)))
    launches = sysm.launch_count() - l0
    t = R.max(float(ms.mean()))
    total = R.sum(float(loss[0]) * (hi - lo))
    t0 = time.perf_counter()
    sysm.lipschitz_loss(Z1l, Z2l)
    e2e_t = R.max(time.perf_counter() - t0)
    # training side: the same loss and its parameter gradient dL/dtheta
    sysm.lipschitz_loss_grad(Z1l[:8], Z2l[:8])
    t0 = time.perf_counter()
    sysm.lipschitz_loss_grad(Z1l, Z2l)
    train_t = R.max(time.perf_counter() - t0)
    hbm, bf16, peak_kind = peaks()
    flops = 890e9 + 640e9  # tangent GEMMs + element HVPs per 1024 pairs
    achieved = flops / (t * 1e-3) / 1e12
    rec = {
        "config": {"workload": f"c5: {Pt} pairs (z1, z2) ~ N(0, 0.25 I) (substream(4,0)) on the c2 problem, full "
                               "16x16 subspace Hessians of the elastic potential at both points (2048 Hessians), "
                               "order-2 loss combined in fp64",
                   "l2": f"flushed before every call ({FLUSH_BYTES >> 20} MiB write)",
                   "parallelism": f"pairs sharded x{R.ws}"},
        "metric": "ms per Lipschitz loss", "value": t, "unit": "ms", "higher_is_better": False,
        "hessians_per_s": 2 * Pt / (t * 1e-3), "loss": total / Pt, "reps": reps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": bf16, "unit": "TFLOP/s",
                     "frac": achieved / bf16, "traffic": None, "algorithmic_flops": flops,
                     "peak_kind": peak_kind + ", dense bf16",
                     "note": "SURVEY 8(d): tangent GEMMs 890 GFLOP + element HVPs 640 GFLOP per 1024 pairs",
                     # the element HVPs alone against the fp32 CUDA-core peak (148 SMs x 128 lanes x 2 x 1.965 GHz)
                     "element_hvp_fp32_frac": 0.64e12 * Pt / 1024 / (t * 1e-3) / (74.4e12 * R.ws)},
        "e2e": {"value": e2e_t * 1e3, "unit": "ms", "h2d_bytes_per_step": 16 * (hi - lo) * r,
                "d2h_bytes_per_step": 8, "api": "lsb_lipschitz_loss (C ABI), host buffers"},
        "gpu_launches": int(launches // reps),
        "timed": "CUDA events on the context stream around each lsb_lipschitz_loss call",
        "train_step_ms": train_t * 1e3,
        "train_step": "lsb_lipschitz_loss_grad over the same pairs (loss + dL/dtheta of every decoder parameter), "
                      "host clock",
    }
    if want_cpu and R.rank == 0 and R.ws == 1:
        ob = oracle_problem("c5")
        sp = 2
        t0 = time.perf_counter()
        lo_cpu = ob.lipschitz_loss2(Z1[:sp], Z2[:sp], threads=1)
        dt = time.perf_counter() - t0
        rec["cpu_baseline"] = {"value": dt * 1e3 / sp * Pt, "unit": "ms", "cores": 1, "kind": "port",
                               "cpu": cpu_model(), "extrapolated": True,
                               "sample": f"{sp} pairs ({2 * sp} Hessians via r(r+1)/2 directional passes, "
                                         f"{dt:.1f} s) on 1 core, scaled to {Pt} pairs",
                               "loss_on_sample": lo_cpu}
    sysm.close()
    return rec


# ------------------------------------------------------------------------------------ reference arm
def run_reference(args, ws, rank):
    """--impl reference: the reference's CPU algorithm (oracle port) on all host cores, on the
    headline workload (E+grad evals of the config's timestep-0 objective)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    per_step = threads
    name = args.config
    oracle_problem(name)  # build outside the timed region
    for _ in range(args.warmup):
        cpu_eval_rate(name, per_step, threads)
    t_all, n_all = 0.0, 0
    for _ in range(args.steps):
        _, dt = cpu_eval_rate(name, per_step, threads)
        t_all += dt
        n_all += per_step
    value = n_all / t_all
    line = {
        "impl": "reference", "metric": "E+grad evals/sec", "value": value, "unit": "evals/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{name}: E+grad evals of the timestep-0 objective, {per_step} seeded z per step",
                   "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port", "cpu": cpu_model(),
                         "sample": f"{args.steps} x {per_step} evals ({name}), oracle C++ -O3 (restatement of the "
                                   "reference, which cannot be built here), std::thread over independent z"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c2f", "c3"])
    ap.add_argument("--records", default="c1,c2,c2f,c4,c5", help="comma list of extra per-config records, or none")
    ap.add_argument("--timesteps", type=int, default=0, help="timesteps for ms/timestep (0: the config's own)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    maybe_relaunch(sys.argv[1:], args.gpus)
    args.warmup = max(args.warmup, 3)
    ws, rank, local, dist = dist_init(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return
    from paper_2409_03807_b200 import configs
    R = Ranks(ws, rank, local, dist)
    K, W = args.steps, args.warmup
    want_cpu = not args.no_cpu_baseline
    cpu_samples = {"c1": 400, "c2": 60, "c2f": 60, "c3": 4}
    with ClockSampler(local) as clk:
        head = single_instance(args.config, K, W, args.timesteps or configs.SPECS[args.config].steps, R, want_cpu,
                               cpu_samples[args.config])
    records = {}
    wanted = [] if args.records in ("", "none") else [x.strip() for x in args.records.split(",")]
    for name in wanted:
        if name == args.config:
            continue
        if name in ("c1", "c2", "c2f", "c3"):
            records[name] = single_instance(name, K, W, args.timesteps or configs.SPECS[name].steps, R, want_cpu,
                                            cpu_samples[name])
        elif name == "c4":
            records[name] = batched_record(K, W, R, want_cpu)
        elif name == "c5":
            records[name] = lipschitz_record(K, W, R, want_cpu)
    if rank == 0:
        line = {
            "metric": "E+grad evals/sec", "value": head["value"], "unit": "evals/s", "n_gpus": ws, "steps": K,
            "warmup": W, "ms_per_step": head["ms_per_eval"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": head["dtype"],
            "data": "synthetic (seeded mesh, Xavier-normal decoder, z ~ N(0, 0.25 I))",
            "config": head["config"],
            "ms_per_timestep": head["timesteps"]["ms_per_timestep"], "timesteps": head["timesteps"],
            "value_only_evals_per_s": head["value_only_evals_per_s"], "clean_l2": head["clean_l2"],
            "roofline": head["roofline"], "cpu_baseline": head.get("cpu_baseline"), "e2e": head["e2e"],
            "clocks": clk.summary(), "gpu_launches": head["gpu_launches"], "energy_check": head["energy_check"],
            "dev_flags": head["dev_flags"], "solve_path": head["solve_path"], "cpu_model": cpu_model(),
            "records": records,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
