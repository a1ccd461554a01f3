#!/usr/bin/env python
"""Benchmark of the B200-native reduced-objective hot path (BASELINE.json metric:
"E+grad evals/sec and ms/timestep (L-BFGS, eps=1e-5); % of HBM roofline").

Workload (N=1 default): BASELINE.json configs[1] = config 2 (16x16x64 Kuhn bar,
98,304 tets, d=16, 5x128 ELU decoder, seed 1), fp64, the timestep-0 objective
E(z) = |f(z) - qbar|_M^2/(2h^2) + P(f(z)).  One bench "step" = one E+grad E
evaluation at a fresh seeded z ~ N(0, 0.5^2 I) (inputs resident in HBM).  Before
every timed step L2 is flushed (a 512 MiB write), so W_out (54 MB fp64) is read
from HBM each step.  ms/timestep of the device-resident L-BFGS (same config,
dynamics from rest) is reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c1|c2|c2f|c3]

Multi-GPU: the single-instance solve does not shard ("replicas
only"): each rank runs an independent replica; value = evals of all ranks /
max-over-ranks time.  --impl reference times the CPU oracle (C++ restatement of
the reference, which cannot be built here) on all host cores, rank 0 only.
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

FLUSH_BYTES = 512 << 20
# dram__bytes_read.sum + dram__bytes_write.sum per launch of the reported kernel, from the
# committed ncu --set full captures (profiles/); None until captured for that path.
TRAFFIC = {
    # profiles/r01_solve_c2_v5_full.txt: one c2 fp64 E+grad eval (ncu flushes caches before the
    # launch, like the bench's L2 flush): dram read 75.42 MB + write 5.79 MB
    ("c2", True): 81.20e6,
}
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(n, h, E, w, per_tet_material=False):
    """Per-eval bytes: w(2nh + 9n) + E(16 + 10w) [+ 2wE]; and the
    output-layer kernel's share: W_out (n h w) + b, s, shift-X, qbar-X, m (5n 8B)
    + u, r written (2n 8B)."""
    total = w * (2 * n * h + 9 * n) + E * (16 + 10 * w) + (2 * w * E if per_tet_material else 0)
    out_fwd = n * h * w + 7 * n * 8
    return total, out_fwd


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


def cpu_eval_rate(name, evals, threads, rng_seed=11):
    """Oracle (C++ restatement, -O3) E+grad evals/s on `threads` host threads."""
    from oracle import pyoracle
    from paper_2409_03807_b200 import configs
    ob = pyoracle.problem(name if name != "c2f" else "c2")
    pr_r = {"c1": 8, "c2": 16, "c2f": 16, "c3": 32}[name]
    X = ob.mesh_arrays()[0]
    free = np.nonzero(ob.mesh_arrays()[4] >= 0)[0]
    qbar = X[free].reshape(-1) + configs.DT ** 2 * np.tile(configs.GRAVITY, free.size)
    Z = 0.5 * np.random.default_rng(rng_seed).standard_normal((evals, pr_r))
    ob.eval_batch(Z[:min(2, evals)], qbar=qbar, dt=configs.DT, threads=1)  # warm
    t0 = time.perf_counter()
    ob.eval_batch(Z, qbar=qbar, dt=configs.DT, threads=threads)
    dt = time.perf_counter() - t0
    return evals / dt, dt


def run_reference(args, ws, rank):
    """--impl reference: the reference's CPU algorithm (oracle port) on all host cores."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    per_step = max(threads, 8)
    rates = []
    for _ in range(args.warmup):
        cpu_eval_rate(args.config, per_step, threads)
    t_all = 0.0
    n_all = 0
    for _ in range(args.steps):
        r, dt = cpu_eval_rate(args.config, per_step, threads)
        rates.append(r)
        t_all += dt
        n_all += per_step
    value = n_all / t_all
    line = {
        "impl": "reference", "metric": "E+grad evals/sec", "value": value, "unit": "evals/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: E+grad evals of the timestep-0 objective, "
                               f"{per_step} seeded z per step", "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} x {per_step} evals ({args.config}), oracle C++ -O3, "
                                   f"std::thread over independent z"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c2f", "c3"])
    ap.add_argument("--timesteps", type=int, default=20, help="timesteps for ms/timestep")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local, dist = dist_init(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        if dist:
            dist.barrier()
        return

    import paper_2409_03807_b200 as P
    from paper_2409_03807_b200 import configs
    pr = configs.build(args.config)
    sysm = pr.system(device=local)
    spec = pr.spec
    n, r, h, E = pr.model.n, pr.model.r, spec.width, pr.mesh.num_elements()
    w = 8 if sysm.precision == "fp64" else 4
    qbar = configs.timestep0_qbar(pr, sysm.mass)
    sysm.set_inertia(qbar, configs.DT)
    K, W = args.steps, args.warmup
    Z = configs.gaussian_latents(100 + rank, K + W, r)
    import ctypes as C
    L = P.lib()

    def bench_evals(Zs):
        k = Zs.shape[0]
        ev = np.zeros(k)
        of = np.zeros(k)
        Es = np.zeros(k)
        P.check(L.lsb_bench_evals(sysm.handle, k, P.dptr(np.ascontiguousarray(Zs)), FLUSH_BYTES, P.dptr(ev),
                                  P.dptr(of), P.dptr(Es)))
        return ev, of, Es

    bench_evals(Z[:W])  # warm-up (untimed)
    if dist:
        dist.barrier()
    launches0 = sysm.launch_count()
    with ClockSampler(local) as clk:
        ev_ms, of_ms, Es = bench_evals(Z[W:])
    launches = sysm.launch_count() - launches0
    t_total_ms = float(ev_ms.sum())
    if dist:
        import torch
        t = torch.tensor([t_total_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_total_ms = float(t.item())
    value = ws * K / (t_total_ms * 1e-3)

    # ---- ms/timestep: device-resident L-BFGS steps from rest (gravity), L2 flushed per step
    st = pr.initial_state()
    sysm.set_state(st)
    sysm.set_external_force(P.gravity_force(pr.mesh, sysm.mass, configs.GRAVITY))
    cfg = configs.solver_config()
    T = max(args.timesteps, 1)
    step_ms = np.zeros(T)
    reps = (P._capi.lsb_exit_report * T)()
    c = cfg._c()
    P.check(L.lsb_bench_steps(sysm.handle, T, C.byref(c), 0, FLUSH_BYTES, P.dptr(step_ms), reps))
    iters = [reps[i].iterations for i in range(T)]
    vevals = [reps[i].value_evals for i in range(T)]
    codes = sorted(set(reps[i].code for i in range(T)))

    # ---- e2e: the reference-facing C-ABI call lsb_eval (host z in, host E and grad out, the
    # copies inside every call), K calls timed on the host clock; and the same through the
    # Python binding (ReducedSystem.eval), reported beside it
    sysm.set_inertia(qbar, configs.DT)
    Ze = np.ascontiguousarray(configs.gaussian_latents(7, K + W, r))
    Ee, Ge = np.zeros(K + W), np.zeros((K + W, r))
    secs = C.c_double()
    P.check(L.lsb_bench_e2e(sysm.handle, W, P.dptr(Ze[:W]), P.dptr(Ee[:W]), P.dptr(Ge[:W]), C.byref(secs)))
    P.check(L.lsb_bench_e2e(sysm.handle, K, P.dptr(np.ascontiguousarray(Ze[W:])), P.dptr(Ee[W:]),
                            P.dptr(Ge[W:]), C.byref(secs)))
    e2e_t = secs.value
    e2e_value = ws * K / e2e_t if e2e_t > 0 else None
    py_t = 0.0
    for k in range(W, W + K):
        t0 = time.perf_counter()
        sysm.eval(Ze[k])
        py_t += time.perf_counter() - t0
    e2e_python = ws * K / py_t if py_t > 0 else None

    # ---- roofline of the dominant kernel
    hbm, peak_kind = peaks()
    alg_total, alg_out = algorithmic_bytes(n, h, E, w, per_tet_material=spec.young[1] > spec.young[0])
    solve = sysm.solve_kernel_info()
    if solve["in_use"]:
        # one persistent launch per evaluation: the kernel IS the evaluation
        kname, alg, dur_s = "solve_kernel (persistent cluster kernel, one launch per eval)", alg_total, float(of_ms.mean()) * 1e-3
    else:
        kname, alg, dur_s = "out_fwd_tma_kernel", alg_out, float(of_ms.mean()) * 1e-3
    achieved = alg / dur_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": TRAFFIC.get((args.config, solve["in_use"])), "kernel": kname, "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": alg,
            "algorithmic_formula": "w(2nh+9n)+E(16+10w)[+2wE] per E+grad eval (SURVEY 8d)" if solve["in_use"]
            else "n h w + 56 n (W_out stream + per-row operands)",
            "solve_grid": solve["grid"],
            "eval_frac": (alg_total / (t_total_ms * 1e-3 / K)) / 1e9 / hbm}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        sample = {"c1": 400, "c2": 120, "c2f": 120, "c3": 4}[args.config]
        rate, dt = cpu_eval_rate(args.config, sample, 1)
        cpu = {"value": rate, "unit": "evals/s", "cores": 1, "kind": "port",
               "sample": f"{sample} E+grad evals of {args.config} on 1 host core (oracle C++ -O3, {dt:.1f} s); "
                         f"the reference is single-threaded"}

    if rank == 0:
        line = {
            "metric": "E+grad evals/sec", "value": value, "unit": "evals/s", "n_gpus": ws, "steps": K,
            "warmup": W, "ms_per_step": t_total_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if w == 8 else "f32 storage / f64 arithmetic",
            "data": "synthetic (seeded mesh, Xavier-normal decoder, z ~ N(0, 0.25 I))",
            "config": {"workload": f"{args.config}: {spec.grid[0]}x{spec.grid[1]}x{spec.grid[2]} Kuhn bar, "
                                   f"{E} tets, n={n}, d={r}, {spec.hidden_layers}x{h} ELU, {sysm.precision}; "
                                   "one E+grad eval per step (timestep-0 objective)",
                       "l2": f"flushed before every timed step ({FLUSH_BYTES >> 20} MiB write)",
                       "parallelism": f"replicas x{ws}"},
            "ms_per_timestep": float(step_ms.mean()), "timesteps": T,
            "timestep_iterations": iters, "timestep_value_evals": vevals, "timestep_codes": codes,
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": 8 * r,
                    "d2h_bytes_per_step": 8 * (1 + r), "api": "lsb_eval (C ABI), host buffers",
                    "python_binding_value": e2e_python},
            "clocks": clk.summary(), "gpu_launches": int(launches),
            "energy_check": float(Es[0]),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
