"""Benchmark: randQB_FP time-to-epsilon on BASELINE config 2 (dense 8000 x 8000,
sigma_j = 1/j, b=50, P=1, eps = 5e-2 relative, max rank 2000, l~ = 2000).

One "step" = one complete rand_qb_fp factorization (Omega generation, the 4 DMMA
passes over A, the wide orthonormalisations of the power step, and the A-free block
loop with the on-device error indicator) until Q, B and the rank are final on the
device. `value` is the device time per step with A resident in HBM (512 MB > L2,
so no L2 flush is needed); `e2e` is the same call through the C-ABI from pinned host
memory: H2D of A, the factorization, and D2H of Q and B every step.

A is the pinned config-2 input of tools/pinned_inputs.py (bit-identical on every x86-64
host; its SHA-256 is in `config`), the same bytes the reference arm and the golden
fixtures use.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one process per GPU, NCCL): config 2 row-sharded over the N ranks
(A, G, Y, Q by rows; the n x l allreduce after each A^T pass and the
Gram allreduces over NCCL), timed max over ranks — strong scaling. Every N also reports
configs 3, 4 and 5 (time-to-eps; the sparse configs with their CSR pass against the HBM
roofline) under `configs`, row-sharded the same way at N > 1.
--impl reference: the reference's own CPU path (oracle/_ref: the reference's kernels,
RNG and containers + the restated rand_qb_fp) run to epsilon on config 2, rank 0 only.
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
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

import pinned_inputs  # noqa: E402

METRIC = "randQB_FP time-to-eps (s), config 2"
CFG = dict(n=8000, b=50, power=1, eps_rel=5e-2, max_rank=2000, l_budget=2000, omega_seed=42)
REF_CACHE = os.path.join(pinned_inputs.CACHE, "ref_arm_cfg2.json")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def workload_config(world: int, sha: str) -> dict:
    """Identical in both arms."""
    return {"workload": "cfg2: randQB_FP dense 8000x8000 sigma_j=1/j, b=50, P=1, eps=5e-2 rel, max rank 2000, "
                        "l~=2000", "n": CFG["n"], "b": CFG["b"], "power": CFG["power"], "eps_rel": CFG["eps_rel"],
            "l_budget": CFG["l_budget"], "max_rank": CFG["max_rank"], "omega_seed": CFG["omega_seed"],
            "a_sha256": sha[:16], "l2": "inputs larger than L2 (A = 512 MB)",
            "parallelism": f"row-sharded x{world}" if world > 1 else "single GPU"}


DATA = ("synthetic (config-2 recipe: A = U diag(1/j) V^T, U,V = Q of QR of RngStream(2) gaussians; "
        "tools/pinned_inputs.py, identical bytes in both arms)")


def host_info() -> dict:
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": model}


# ---- clocks ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if "Active" in r[4 + i] and "Not" not in r[4 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---- reference CPU arm -------------------------------------------------------------------
def reference_time_to_eps(a, sha: str) -> dict:
    """The reference's own CPU path to epsilon on config 2: rand_qb_fp (restated algorithm
    layer, oracle/qb_restated.cpp) over the reference's MatrixHandle / DenseMatrix /
    gemm_nn / gemm_tn (kernels_drivers.cpp:21-65, AVX2 lane) and RngStream (rng.cpp),
    compiled from /root/reference/proj/src into oracle/_ref/libqbref.so. The time is the
    oracle's steady_clock around the rand_qb_fp call (matrix wrap excluded). One core:
    the reference has no threads."""
    from oracle import oracle as O

    a = np.asfortranarray(a)
    eps = CFG["eps_rel"] * float(np.linalg.norm(a))
    r = O.run("fp", a, b=CFG["b"], power=CFG["power"], eps_abs=eps, l_budget=CFG["l_budget"],
              max_rank=CFG["max_rank"], seed=CFG["omega_seed"])
    out = {"value": r.seconds, "rank": r.rank, "passes": r.passes, "terminated_by": r.terminated_by,
           "E": r.E, "lane": O.lane_name(), "a_sha256": sha, "host": host_info(),
           "when": time.strftime("%Y-%m-%dT%H:%M:%S")}
    os.makedirs(os.path.dirname(REF_CACHE), exist_ok=True)
    json.dump(out, open(REF_CACHE, "w"))
    return out


def cpu_baseline_obj(ref: dict, how: str) -> dict:
    return {"value": ref["value"], "unit": "s", "cores": 1, "kind": "reference",
            "sample": f"full reference rand_qb_fp to eps on config 2 (lane {ref['lane']}, rank {ref['rank']}, "
                      f"{ref['passes']} passes, {ref['terminated_by']}), one core of {ref['host']['cpu']} "
                      f"({ref['host']['nproc']} cores); {how}"}


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    a, sha = pinned_inputs.matrix(2, gauss="oracle")  # no library of this repo is loaded on this arm
    steps = max(1, min(args.steps, env_int("QBFAC_REF_STEPS", 1)))
    times, last = [], None
    for _ in range(steps):
        last = reference_time_to_eps(a, sha)
        times.append(last["value"])
    v = float(np.median(times))
    last["value"] = v
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": steps,
            "steps_requested": args.steps, "warmup": 0, "warmup_requested": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "impl": "reference", "config": workload_config(args.gpus, sha),
            "result": {"rank": last["rank"], "passes": last["passes"], "terminated_by": last["terminated_by"]},
            "cpu_baseline": cpu_baseline_obj(last, f"{steps} full run(s), warm-up skipped (a run is ~3 min)"),
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm -------------------------------------------------------------------------------
class Dist:
    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
        torch.cuda.set_device(self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t)
        return float(t.item())


def timed_device(ctx, fn, steps):
    import torch
    stream = torch.cuda.ExternalStream(ctx.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    ctx.synchronize()
    return e0.elapsed_time(e1) / 1e3 / steps


def hbm_peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 7700.0  # B200_PROFILING.md fallback


def time_config(D, ctx, h, run, steps):
    """Device time per run (CUDA events on the library stream, max over ranks) after one warm run;
    also the per-run wall times and the SM clock during the runs."""
    r = run()
    info = qbfac_info(r)
    r.free()
    ctx.synchronize()
    D.barrier()
    clocks = ClockSampler(D.local)
    clocks.start()
    time.sleep(0.2)
    walls = []

    def one():
        t0 = time.perf_counter()
        x = run()
        x.free()
        ctx.synchronize()
        walls.append(time.perf_counter() - t0)
    t = timed_device(ctx, one, steps)
    info["run_wall_s"] = [round(w, 5) for w in walls]
    info["clocks"] = clocks.stop()
    return D.max(t), info


def qbfac_info(r):
    from paper_1606_09402_b200 import qbfac
    i = qbfac.info_dict(r.info)
    return {"rank": int(i["rank"]), "passes": int(i["passes"]), "blocks": int(i["blocks"]),
            "terminated_by": qbfac.TERMINATION[int(i["terminated_by"])]}


def config_dense4(D, ctx, steps=3):
    """Config 4 (single-pass FP, 40000 x 20000, l = 400, b = 100), row-sharded over the ranks at
    N > 1: G = A_g Omega local, H = sum_g A_g^T G_g allreduced once (64 MB), Grams allreduced."""
    import torch

    from paper_1606_09402_b200 import dist as qdist
    from paper_1606_09402_b200 import matgen, qbfac
    m, n, w = 40000, 20000, 400
    row0, rows = qdist.plan_dense_rows(m, D.world)[D.rank]
    sig = np.exp(-np.arange(1, 401) / 60.0)
    at = matgen.synthesize_torch(m, n, sig, 4, noise=1e-6)  # device-synthesized (timing only)
    a_loc = at.t()[row0:row0 + rows].cpu().numpy()
    del at
    torch.cuda.empty_cache()
    h = qbfac.MatrixHandle.dense_shard(a_loc, m, row0, ctx) if D.world > 1 else qbfac.MatrixHandle.dense(a_loc, ctx)
    del a_loc
    t, info = time_config(D, ctx, h, lambda: qbfac.run_device(h, alg=3, mode=0, b=100, power=0, k=w, s=0, seed=42),
                          steps)
    pt = pass_time(h, w, False, ctx)
    out = {"workload": "cfg4: single-pass FP 40000x20000 rank-400 + 1e-6 noise, l=400, b=100 (device-synthesized A)",
           "time_to_eps_s": t, **info, "rows_per_rank": rows, "pass_nn_ms_local": pt * 1e3,
           "pass_nn_tflops_local": 2.0 * rows * n * w / pt / 1e12}
    h.free()
    return out


def config_sparse(D, ctx, cfg, steps=2):
    """Config 3 (EI CSR 1e5 x 5e4, 5M nnz, b=50, P=1) or 5 (EI CSR 2e6 x 5e5 Zipf, 2e8 nnz,
    b=100, P=2), rows balanced by nnz over the ranks at N > 1. Reports time-to-eps and the
    CSR pass A*X at width b against the HBM roofline (algorithmic bytes 12 nnz + 8 (rows + 1)
    + 8 (n + rows) w: A, X and Y once)."""
    from paper_1606_09402_b200 import dist as qdist
    from paper_1606_09402_b200 import matgen, qbfac
    if cfg == 3:
        csr, b, power, eps_rel, cap = matgen.csr_uniform(100000, 50000, 50, seed=3), 50, 1, 0.5, 1000
        wl = "cfg3: EI CSR 1e5x5e4, 5M nnz uniform, b=50, P=1, eps=0.5 rel, cap 1000"
    else:
        csr, b, power, eps_rel, cap = matgen.csr_zipf(2_000_000, 500_000, alpha=1.1, target_nnz=2e8, seed=5), 100, 2, 0.6, 2000
        wl = "cfg5: EI CSR 2e6x5e5 Zipf(1.1), 2e8 nnz, b=100, P=2, eps=0.6 rel, cap 2000"
    m, n = csr[0], csr[1]
    row0, rows = qdist.plan_csr_rows(csr[2], D.world)[D.rank]
    _, _, rp, ci, v = qdist.shard_csr(csr, row0, rows)
    norm = float(np.sqrt(D.sum(float(v @ v))))
    h = (qbfac.MatrixHandle.csr_shard(m, row0, n, rp, ci, v, ctx) if D.world > 1
         else qbfac.MatrixHandle.csr(m, n, rp, ci, v, ctx))
    nnz = len(v)
    del csr
    t, info = time_config(D, ctx, h, lambda: qbfac.run_device(h, alg=0, b=b, power=power, max_rank=cap,
                                                                eps_abs=eps_rel * norm, seed=42), steps)
    pt = pass_time(h, b, False, ctx)
    alg_bytes = 12.0 * nnz + 8.0 * (rows + 1) + 8.0 * (n + rows) * b
    out = {"workload": wl, "time_to_eps_s": t, **info, "nnz_local": int(nnz), "rows_per_rank": rows,
           "pass_n_ms_local": pt * 1e3, "pass_n_alg_gbs": alg_bytes / pt / 1e9,
           "pass_n_frac_hbm": alg_bytes / pt / 1e9 / hbm_peak_gbs()}
    h.free()
    return out


def pass_time(h, w, trans, ctx, reps=5):
    import torch
    rows_in = h.m if trans else h.n
    rows_out = h.n if trans else h.m
    x = torch.randn((rows_in, w), dtype=torch.float64, device="cuda")
    y = torch.empty((rows_out, w), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):
        h.multiply_device(x.data_ptr(), w, w, trans, y.data_ptr(), w)
    ctx.synchronize()
    return timed_device(ctx, lambda: h.multiply_device(x.data_ptr(), w, w, trans, y.data_ptr(), w), reps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the config 3/4/5 sub-measurements")
    ap.add_argument("--no-cfg5", action="store_true", help="skip config 5 (2e8 nnz; ~1 min to generate)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    D = Dist()
    torch = D.torch
    from paper_1606_09402_b200 import dist as qdist
    from paper_1606_09402_b200 import qbfac

    # the pinned input: built once (local rank 0), then every rank maps the same file
    if D.local == 0:
        pinned_inputs.matrix(2)
    D.barrier()
    a_host, sha = pinned_inputs.matrix(2)
    n = CFG["n"]
    eps = CFG["eps_rel"] * float(np.linalg.norm(np.asfortranarray(a_host)))
    os.environ["QBFAC_DEVICE"] = str(D.local)
    if D.world > 1:
        ctx = qdist.sharded_context(D.local)
        row0, rows = qdist.plan_dense_rows(n, D.world)[D.rank]
        a_loc = np.asfortranarray(a_host[row0:row0 + rows])
        handle = qbfac.MatrixHandle.dense_shard(a_loc, n, row0, ctx)
    else:
        ctx = qbfac.Context(D.local)
        row0, rows = 0, n
        a_loc = np.asfortranarray(a_host)
        handle = qbfac.MatrixHandle.dense(a_loc, ctx)

    def factorize(h=handle):
        return qbfac.run_device(h, alg=1, b=CFG["b"], power=CFG["power"], max_rank=CFG["max_rank"],
                                l_budget=CFG["l_budget"], eps_abs=eps, seed=CFG["omega_seed"])

    for _ in range(args.warmup):
        r = factorize()
        info = qbfac.info_dict(r.info)
        r.free()
    ctx.synchronize()

    # ---- timed region: A (this rank's rows) resident in HBM ----
    clocks = ClockSampler(D.local)
    clocks.start()
    time.sleep(0.2)
    D.barrier()
    ctx.synchronize()
    l0 = ctx.kernel_launches()
    # each result is released right away (stream-ordered free: no sync); results kept alive across
    # the timed runs would grow the memory pool inside the timed region
    t_step = timed_device(ctx, lambda: factorize().free(), args.steps)
    D.barrier()
    launches = ctx.kernel_launches() - l0
    clk = clocks.stop()
    t_step = D.max(t_step)

    # ---- e2e: through the C-ABI from pinned host memory, Q and B back to the host ----
    host_a = torch.empty((a_loc.shape[1], a_loc.shape[0]), dtype=torch.float64, pin_memory=True)
    host_a.numpy()[:] = a_loc.T
    a_view = host_a.numpy().T  # column-major rows x n, pinned
    q_out = torch.empty(rows * CFG["max_rank"], dtype=torch.float64, pin_memory=True).numpy()
    b_out = torch.empty(n * CFG["max_rank"], dtype=torch.float64, pin_memory=True).numpy()
    e2e_times, h2d, d2h, phases = [], 0, 0, []
    for s in range(max(2, min(args.steps, 5))):
        ctx.synchronize()
        D.barrier()
        t0 = time.perf_counter()
        if D.world > 1:
            h = qbfac.MatrixHandle.dense_shard(a_view, n, row0, ctx)  # H2D of this rank's rows
        else:
            # H2D in row chunks on the copy stream; the first pass G = A*Omega consumes each
            # chunk as it lands (qbfac_gpu_matrix_dense_async)
            h = qbfac.MatrixHandle.dense_async(a_view, ctx)
        t1 = time.perf_counter()
        r = factorize(h)
        t2 = time.perf_counter()
        q = r.q(q_out)                                      # D2H of Q (this rank's rows)
        b = r.b(b_out) if D.rank == 0 else np.zeros(0)      # D2H of B (replicated: rank 0)
        t3 = time.perf_counter()
        r.free()
        h.free()
        ctx.synchronize()
        e2e_times.append(time.perf_counter() - t0)
        phases.append((t1 - t0, t2 - t1, t3 - t2, e2e_times[-1] - (t3 - t0)))
        h2d = int(D.sum(8.0 * a_view.size))
        d2h = int(D.sum(8.0 * (q.size + b.size)))
    t_e2e = D.max(float(np.median(e2e_times)))
    ph = np.median(np.array(phases), axis=0) * 1e3
    e2e_extra = {"phases_ms": {"handle": round(float(ph[0]), 3), "run": round(float(ph[1]), 3),
                               "d2h_q_b": round(float(ph[2]), 3), "free_sync": round(float(ph[3]), 3)},
                 "all_s": [round(t, 5) for t in e2e_times]}
    if D.world == 1:
        dev_a = torch.empty_like(host_a, device="cuda")
        h2d_s = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev_a.copy_(host_a, non_blocking=True)
            torch.cuda.synchronize()
            h2d_s.append(time.perf_counter() - t0)
        del dev_a
        e2e_extra["h2d_link_gbs"] = round(8 * host_a.numel() / min(h2d_s) / 1e9, 2)

    # ---- roofline: the dominant kernel (DMMA pass G = A * Omega at width l~, this rank's rows) ----
    w = CFG["l_budget"]
    t_pass = pass_time(handle, w, False, ctx)
    t_pass_t = pass_time(handle, w, True, ctx)
    flops = 2.0 * rows * n * w
    achieved = flops / t_pass / 1e12
    pa = torch.randn((8192, 8192), dtype=torch.float64, device="cuda")
    pb = torch.randn((8192, 8192), dtype=torch.float64, device="cuda")
    pa @ pb
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        pa @ pb
        c1.record()
        torch.cuda.synchronize()
        best = min(best, c0.elapsed_time(c1) / 1e3)
    peak = 2 * 8192**3 / best / 1e12
    del pa, pb
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and D.world == 1:
        try:
            traffic = json.load(open(tpath)).get("dense_pass_nn_per_launch_bytes")
        except Exception:
            traffic = None
    comm = None
    if D.world > 1:
        # the n x l~ allreduce of H = A^T G (the pass's only collective), timed the same way
        buf = torch.ones((n * w,), dtype=torch.float64, device="cuda")
        for _ in range(2):
            D.dist.all_reduce(buf)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(5):
            D.dist.all_reduce(buf)
        c1.record()
        torch.cuda.synchronize()
        ar = D.max(c0.elapsed_time(c1) / 5 / 1e3)
        comm = {"allreduce_n_x_l_ms": ar * 1e3, "bytes": 8 * n * w, "busbw_gbs": 2 * (D.world - 1) / D.world * 8 * n * w / ar / 1e9}
        del buf

    configs = {}
    if not args.no_configs:
        handle.free()
        torch.cuda.empty_cache()
        configs["cfg3"] = config_sparse(D, ctx, 3)
        configs["cfg4"] = config_dense4(D, ctx)
        if not args.no_cfg5:
            configs["cfg5"] = config_sparse(D, ctx, 5)

    cpu = None
    if D.rank == 0 and D.world == 1 and not args.no_cpu_baseline:
        try:
            ref = json.load(open(REF_CACHE)) if os.path.exists(REF_CACHE) else None
            if ref and ref.get("a_sha256") == sha:
                cpu = cpu_baseline_obj(ref, f"measured by bench.py --impl reference on this host at {ref['when']}")
            else:
                ref = reference_time_to_eps(a_host, sha)
                cpu = cpu_baseline_obj(ref, "measured in this run")
        except Exception as ex:  # the oracle is a reported baseline, never the product path
            cpu = {"value": None, "unit": "s", "cores": 1, "kind": "reference", "sample": f"unavailable: {ex}"}

    if D.rank == 0:
        line = {
            "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": D.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": workload_config(D.world, sha),
            "result": {"rank": info["rank"], "passes": info["passes"], "blocks": info["blocks"],
                       "terminated_by": qbfac.TERMINATION[int(info["terminated_by"])],
                       "householder_fallbacks": info["householder_fallbacks"], "rows_per_rank": rows},
            "clocks": clk,
            "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, **e2e_extra},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"dgemm_ws_kernel (DMMA, TMA + mbarrier ring) G = A*Omega, {rows}x{n}x{w}",
                         "peak_source": "cuBLAS DGEMM 8192^3 measured live in this run (FP64 tensor; "
                                        "MEASURED_PEAKS.json has no FP64 entry)",
                         "pass_nn_ms": t_pass * 1e3, "pass_tn_ms": t_pass_t * 1e3,
                         "pass_tn_tflops": flops / t_pass_t / 1e12},
            "comm": comm,
            "configs": configs or None,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if D.world > 1:
        D.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
