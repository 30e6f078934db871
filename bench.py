#!/usr/bin/env python
"""Benchmark of the SuperVoxHenry B200 hot path (BASELINE.json metric:
"FFT-circulant matvec voxel-unknowns/s & % HBM roofline; time to port L-matrix").

One step = one svh_matvec (Eq. 9, all five passes A-E of DESIGN.md) over a
batch of R right-hand sides (one per port) on the workload's full grid.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--nrhs R]
  python bench.py --impl reference ...   # the fp64 CPU oracle on the same workload

Rank 0 prints ONE JSON line.  Under torchrun each rank processes its own R
RHS (weak scaling: independent port excitations, no data-path collective);
timing is CUDA events on the launching stream, max over ranks.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import svh_inputs  # noqa: E402

METRIC = "FFT-circulant matvec voxel-unknowns/s"
UNIT = "voxel-unknowns/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


# BASELINE.json configs[4], the largest single-GPU configuration: the
# 1024 x 1024 x 64 grid (embedding 2048 x 2048 x 128), 50 % Bernoulli fill (seed 5), Tucker
# kernels (tol 1e-4: ranks 4-32 as configs[4] asks, max rank 15), 8 RHS per GPU.
DEFAULT_WORKLOAD = "cfg5"
DEFAULT_TUCKER = {"cfg5": 1e-4}


def workload(name):
    if name == "cfg5":
        c = svh_inputs.random_fill((1024, 1024, 64), fill=0.5, seed=5)
        return dict(c, name="cfg5_fill0.5_1024x1024x64_s5"), 8
    if name == "cfg4":
        return svh_inputs.config4(), 16
    if name == "cfg3":
        return svh_inputs.config3(), 2
    if name == "cfg2":
        c = svh_inputs.config2()
        c = dict(c, tucker_tol=0.0)
        return c, 1
    if name.startswith("fill"):
        # e.g. fill512x512x64
        dims = tuple(int(v) for v in name[4:].split("x"))
        return svh_inputs.random_fill(dims, fill=0.5, seed=5), 4
    raise SystemExit(f"unknown workload {name}")


def bind_to_gpu_numa(index):
    """Run this process on the CPUs local to the GPU's PCIe root (sysfs local_cpulist), so the
    pinned host buffers of the e2e measurement are first-touched on the GPU's NUMA node (a remote
    node costs PCIe bandwidth).  Best effort: returns the cpulist used, or None."""
    try:
        bus = subprocess.run(["nvidia-smi", "-i", str(index), "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=20).stdout.strip().lower()
        dom, rest = bus.split(":", 1)
        path = f"/sys/bus/pci/devices/{dom[-4:]}:{rest}/local_cpulist"
        spec = open(path).read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        os.sched_setaffinity(0, cpus)
        return spec
    except Exception:
        return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region, in-process through NVML
    (pynvml) every 200 ms.  An nvidia-smi child polling at 100 ms was measured to stall the
    launch path of the timed loop by up to ~10 ms per step on this driver; in-process NVML
    queries at a lower rate do not.  Falls back to an nvidia-smi child if NVML is missing."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index, period=0.2):
        self.index, self.period = index, period
        self.rows = []          # (sm_mhz, max_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.t = None

    def _loop(self, nv, hdl):
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(hdl, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(hdl)
                self.rows.append((float(sm), float(mx), int(rs)))
            except Exception:
                pass
            self.stop.wait(self.period)

    def __enter__(self):
        if os.environ.get("SVH_NO_CLOCKS"):
            return self
        try:
            import pynvml as nv
            nv.nvmlInit()
            hdl = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.t = threading.Thread(target=self._loop, args=(nv, hdl), daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        import pynvml as nv
        reasons = sorted(n for n, c in self.REASONS.items() if any(r[2] & getattr(nv, c) for r in self.rows))
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": "NVML in-process, 200 ms"}


def pass_bytes(h, R, packed=True):
    """Algorithmic HBM bytes of each pass per launch (R RHS), DESIGN.md §5.

    Rows (y, z) / planes z holding no voxel are zero in every embedded current and the
    pruned passes never touch them, so with Rn non-empty rows and Pn non-empty planes
    (pts/comp): A reads K (packed) + writes Rn*Nx; B Rn*Nx -> Pn*Ny*Nx; C Pn*Ny*Nx ->
    Pn*Ny*Nx (+ the 7 fp32 octant spectra once, dense mode); D Pn*Ny*Nx -> Rn*Nx;
    E Rn*Nx + K (I again) -> K.  Maps: the row-occupancy words (8 B per 32 cells) and the
    row list (4 B per row) in A and E, the packed material ids (1 B per voxel) in E,
    the row mask in B/D -- each counted once per launch (compulsory bytes).
    """
    kz, ky, kx = h.shape
    K = h.K
    nx, ny, nz = h.embedding
    c8 = 5 * 8 * R
    X1 = h.rows_nonempty * nx
    X2 = h.planes_nonempty * ny * nx
    spec = 7 * 4 * (nx // 2 + 1) * (ny // 2 + 1) * (nz // 2 + 1)
    rowinfo = 8 * h.rows_nonempty * ((kx + 31) // 32) + 4 * h.rows_nonempty
    A = c8 * (K + X1) + rowinfo
    B = c8 * (X1 + X2)
    C = c8 * 2 * X2 + (0 if h.tucker else spec)
    D = c8 * (X2 + X1)
    E = c8 * (X1 + 2 * K) + rowinfo + K
    return [A, B, C, D, E]


def p3s_bytes(h, case, R):
    """Algorithmic HBM bytes of one plan-P3s product, R RHS: A3 reads K (packed)
    and writes Nx*Ry; YZ reads and writes Nx*Ry (+ the octant spectra once, dense mode); E3
    reads Nx*Ry + K (I again) and writes K.  Ry = rows of the live TY-row blocks (TY = 16 for
    Nx = 1024, else 32) of the non-empty planes -- the pruning granularity of the plan."""
    mat = case["mat_id"] != 0
    kz, ky, kx = mat.shape
    nx, ny, nz = h.embedding
    ty = 16 if nx >= 1024 else 32
    rows = mat.any(axis=2)                      # (kz, ky)
    Ry = 0
    for z in range(kz):
        for b in range(0, ky, ty):
            if rows[z, b:b + ty].any():
                Ry += min(ty, ky - b)
    c8 = 5 * 8 * R
    K = h.K
    spec = 7 * 4 * (nx // 2 + 1) * (ny // 2 + 1) * (nz // 2 + 1)
    rowinfo = 8 * h.rows_nonempty * ((kx + 31) // 32)
    A3 = c8 * (K + nx * Ry) + rowinfo
    YZ = c8 * 2 * nx * Ry + (0 if h.tucker else spec)
    E3 = c8 * (nx * Ry + 2 * K) + rowinfo + K
    return [A3, YZ, E3]


def thin_grid_plans(local, name="cfg3", nrhs=(2, 16), steps=20):
    """Plan P5 vs plan P3s on a thin grid, each forced, device-timed with CUDA
    events (inputs resident, 3 warm-up products), with the auto selection's choice."""
    import torch
    from paper_2105_08627_b200 import svh
    case, _ = workload(name)
    peaks, _ = load_peaks()
    out = {"workload": case["name"]}
    for R in nrhs:
        rec = {}
        for plan in (5, 3):
            with svh.setup_case(case, device=local, plan=plan) as h:
                I = torch.from_numpy(svh_inputs.currents(h.K, R, seed=7).astype(np.complex64)).cuda()
                o = torch.empty_like(I)
                for _ in range(3):
                    h.matvec(I, out=o)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(steps):
                    h.matvec(I, out=o)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / steps
                b = sum(pass_bytes(h, R)) if plan == 5 else sum(p3s_bytes(h, case, R))
                kz, ky, kx = h.shape
                rec["P5" if plan == 5 else "P3s"] = {
                    "ms": round(ms, 4), "voxel_unknowns_per_s": 5.0 * kx * ky * kz * R / (ms / 1e3),
                    "bytes": int(b), "frac": round(b / (ms / 1e3) / 1e9 / float(peaks["hbm_gbs"]), 4)}
                del I, o
        with svh.setup_case(case, device=local, plan=0) as h:
            I = torch.from_numpy(svh_inputs.currents(h.K, R, seed=7).astype(np.complex64)).cuda()
            h.matvec(I)
            torch.cuda.synchronize()
            rec["auto_choice"] = "P3s" if h.matvec_plan()[0] == 3 else "P5"
            del I
        torch.cuda.empty_cache()
        out["nrhs_%d" % R] = rec
    return out


def oracle_sample_step(case, frac, seed):
    """One bounded oracle sample: a seeded random fraction `frac` of the source voxels (the
    sub-lattice keeps their positions and materials), one random output voxel (all 5
    components) by the oracle's direct Green sum over those sources.  Returns (seconds,
    number of sources)."""
    from oracle.lattice import Lattice
    from oracle.operator import matvec_direct
    mat = case["mat_id"]
    occ = np.flatnonzero(mat.reshape(-1))
    K = occ.size
    gs = np.random.default_rng(seed)
    keep = np.sort(gs.choice(K, max(1, int(round(frac * K))), replace=False))
    sub = np.zeros(mat.size, dtype=mat.dtype)
    sub[occ[keep]] = mat.reshape(-1)[occ[keep]]
    lat = Lattice(sub.reshape(mat.shape))
    I = svh_inputs.currents(lat.K, 1, seed=seed)
    row = gs.choice(lat.K, 1)
    t0 = time.perf_counter()
    matvec_direct(lat, case["materials"], 2 * np.pi * case["freq"], case["dx"], I, rows=row)
    return time.perf_counter() - t0, lat.K


def cpu_oracle_rate(case, budget_s=20.0, seed=0):
    """Oracle (fp64 direct sum, numpy, as it stands) on a bounded sample of the workload:
    output voxels against a seeded random subset of the sources, the subset sized from a
    calibration step so the timed samples take about budget_s; the per-output-voxel time is
    extrapolated to all K sources and all K outputs (one full 1-RHS matvec).
    Returns (voxel-unknowns/s, seconds, cores, description)."""
    K = int(np.count_nonzero(case["mat_id"]))
    t_cal, n_cal = oracle_sample_step(case, min(1.0, 2000.0 / K), seed + 1)
    per_src = t_cal / n_cal
    frac = min(1.0, budget_s / 4 / (per_src * K))
    times, ns = [], []
    for k in range(4):
        dt, n = oracle_sample_step(case, frac, seed + 10 + k)
        times.append(dt)
        ns.append(n)
    t_row = sum(times) / sum(ns) * K                    # one output voxel against all K sources
    Kt = int(np.prod(case["mat_id"].shape))
    desc = (f"4 sampled output voxels of {case['name']}, each by the fp64 direct sum over a seeded random "
            f"{frac:.2e} of the {K} sources ({sum(times):.1f} s), extrapolated to one full 1-RHS matvec")
    return 5 * Kt / (t_row * K), sum(times), os.cpu_count(), desc


def run_reference(args):
    """--impl reference: the fp64 CPU oracle timed on the host cores (rank 0 only).

    One step = one sampled output voxel (all 5 components) of the workload, summed by the
    oracle's direct Green sum over a seeded random subset of the source voxels; the subset is
    sized once (from a calibration run) so that the whole warm-up + steps run takes about
    2.5 minutes, and the rate is extrapolated to a full 1-RHS matvec (x K / |subset| per row,
    x K rows).  The oracle itself is run as it stands.
    """
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    case, R = workload(args.workload)
    mat = case["mat_id"]
    K = int(np.count_nonzero(mat))
    g = np.random.default_rng(1)

    def sample_step(frac, seed):
        return oracle_sample_step(case, frac, seed)

    t_cal, n_cal = sample_step(min(1.0, 2000.0 / K), 12345)
    budget = 150.0
    frac = min(1.0, budget / max(1, args.warmup + args.steps) / (t_cal * K / n_cal))
    times, ns = [], []
    for st in range(args.warmup + args.steps):
        dt, n = sample_step(frac, int(g.integers(1 << 30)))
        if st >= args.warmup:
            times.append(dt)
            ns.append(n)
    Kt = int(np.prod(mat.shape))
    t_row = float(np.mean(times)) * K / float(np.mean(ns))   # one output voxel against all K sources
    value = 5 * Kt / (t_row * K)          # extrapolated full-matvec rate, 1 RHS
    ms_step = float(np.mean(times)) * 1e3
    sample = (f"{args.steps} steps; each = 1 sampled output voxel (5 components) by the oracle's direct sum over "
              f"a seeded random {frac:.4f} of the {K} source voxels of {case['name']}; rate extrapolated to a full "
              f"1-RHS matvec")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": case["name"], "nrhs": 1, "grid": list(mat.shape[::-1]), "K": K,
                       "source_fraction": frac, "step": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cufft_reference(h, case, R, reps=3):
    """cuFFT reference pipeline (north star: 'cuFFT timed alongside as a reference point,
    not the product'): zero-pad each component to the embedding, torch.fft.fftn (cuFFT),
    5->5 MAC with the 7 full-grid kernel spectra (built from libsvh's kernel tables by
    embedding + cuFFT, outside the timed region), ifftn, crop.  Grid layout, c64.
    Returns ms per RHS."""
    import torch
    kz, ky, kx = h.shape
    nx, ny, nz = h.embedding
    occ = torch.from_numpy(case["mat_id"] != 0).cuda()
    gen = torch.Generator(device="cuda").manual_seed(7)
    I = torch.randn((5, kz, ky, kx), dtype=torch.complex64, device="cuda", generator=gen) * occ
    ours = h.matvec_grid(I[None], green_only=True)[0]   # before the full-grid spectra take the memory
    K = torch.from_numpy(h.kernels()).cuda()            # fp64 [7][kz][ky][kx], m >= 0
    odd = [None, 2, 1, 0, None, None, None]             # K1x odd along x (tensor dim 2), ...
    spec = []
    for q in range(7):
        e = torch.zeros((nz, ny, nx), dtype=torch.float64, device="cuda")
        for sz in (1, -1):
            for sy in (1, -1):
                for sx in (1, -1):
                    sign = 1.0
                    if odd[q] is not None and (sx, sy, sz)[2 - odd[q]] < 0:
                        sign = -1.0
                    zi = torch.arange(kz, device="cuda") * sz % nz
                    yi = torch.arange(ky, device="cuda") * sy % ny
                    xi = torch.arange(kx, device="cuda") * sx % nx
                    e[zi[:, None, None], yi[None, :, None], xi[None, None, :]] = sign * K[q]
        spec.append(torch.fft.fftn(e).to(torch.complex64))
    w = 2 * np.pi * case["freq"]
    g = 1j * w * 4e-7 * np.pi * case["dx"]
    del K

    def one():
        # component by component so the 2048^2 x 128 embedding fits next to the 7 spectra
        Ih = torch.fft.fftn(torch.nn.functional.pad(I, (0, nx - kx, 0, ny - ky, 0, nz - kz)), dim=(1, 2, 3))
        res = torch.empty((5, kz, ky, kx), dtype=torch.complex64, device="cuda")
        P1 = []
        for c in range(3):
            m1 = Ih[3] + Ih[4] if c == 0 else (Ih[4] - Ih[3] if c == 1 else -2 * Ih[4])
            res[c] = (g * torch.fft.ifftn(spec[0] * Ih[c] + spec[1 + c] * m1))[:kz, :ky, :kx]
            P1.append(-spec[1 + c] * Ih[c] + spec[4 + c] * m1)
            del m1
        del Ih
        res[3] = (g * torch.fft.ifftn(P1[0] - P1[1]))[:kz, :ky, :kx]
        res[4] = (g * torch.fft.ifftn(P1[0] + P1[1] - 2 * P1[2]))[:kz, :ky, :kx]
        return res
    ref = one()
    rel = float(torch.linalg.norm((ref - ours)[:, occ]) / torch.linalg.norm(ours[:, occ]))
    del ref, ours
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        one()
    e1.record()
    torch.cuda.synchronize()
    del spec, I, occ
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / reps, rel


def time_to_L(name, device, world, rank):
    """Time to the port L-matrix (BASELINE metric, 3rd part): svh_setup + svh_solve on a
    BASELINE config, wall clock around the public API calls (ports sharded over ranks)."""
    import torch
    from paper_2105_08627_b200 import parallel, svh
    case = {"cfg1": svh_inputs.config1, "cfg2": svh_inputs.config2, "cfg3": svh_inputs.config3,
            "cfg4": svh_inputs.config4}[name]()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inner_tol = 1e-3
    h = svh.setup_case(case, tucker_tol=0.0, device=device, inner_tol=inner_tol)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if world > 1:
        res = parallel.solve_sharded(h, case["ports"])
    else:
        res = h.solve(case["ports"])
    t2 = time.perf_counter()
    h.close()
    st = res["stats"]
    return {"workload": case["name"], "seconds": round(t2 - t0, 4), "setup_s": round(t1 - t0, 4),
            "solve_s": round(t2 - t1, 4), "n_ports": len(case["ports"]),
            "L_pH_diag": [round(float(v) * 1e12, 6) for v in np.diag(res["L"])],
            "gmres_iterations": st.get("total_iterations"), "inner_pcg_iterations": st.get("inner_iterations"),
            "rre": st.get("final_rre"), "converged": st.get("converged"),
            "inner_tol": inner_tol, "rre_target": 1e-6,
            "note": "Schur-complement inner PCG tolerance 1e-3 (the paper's AGMG uses 1e-8, P:166)"}


def run_slab(args, case, R, world, rank, local):
    """--slab: the slab-decomposed matvec, strong scaling (total grid fixed; value = 5 Kt R / t)."""
    import torch
    import torch.distributed as dist
    from paper_2105_08627_b200 import svh
    from paper_2105_08627_b200.parallel import SlabMatvec
    h = svh.setup_case(case, device=local)
    kz, ky, kx = h.shape
    Kt = kx * ky * kz
    P = world if world > 1 else args.slab
    sm = SlabMatvec(h, P, rank=rank if world > 1 else 0)
    g = torch.Generator(device="cuda").manual_seed(100)
    occ = torch.from_numpy(case["mat_id"] != 0).cuda()
    I = (torch.randn((R, 5, kz, ky, kx), dtype=torch.complex64, device="cuda", generator=g) * occ)
    if world > 1:
        I = I[:, :, :, rank * sm.Kyl:(rank + 1) * sm.Kyl, :].contiguous()
    step = (lambda: sm.matvec(I)) if world > 1 else (lambda: sm.matvec_virtual(I))
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    line = {"metric": METRIC, "value": 5.0 * Kt * R / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": {"workload": case["name"], "grid": [kx, ky, kz], "nrhs": R, "slabs": P,
                       "mode": "NCCL all_to_all" if world > 1 else "virtual slabs on one GPU (exchange by copies)",
                       "layout": "grid [nrhs][5][Kz][Ky/P][Kx] per slab"},
            "clocks": clk.summary()}
    h.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--nrhs", type=int, default=0)
    ap.add_argument("--tucker", type=float, default=None,
                    help="Tucker tol (0 = dense octant spectra); default: the workload's (cfg5: 1e-4)")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-solve", action="store_true", help="skip the time-to-L measurement")
    ap.add_argument("--no-cufft", action="store_true", help="skip the cuFFT reference-pipeline timing")
    ap.add_argument("--no-plans", action="store_true", help="skip the thin-grid P5 vs P3s plan comparison")
    ap.add_argument("--solve-workload", default="cfg3")
    ap.add_argument("--slab", type=int, default=0,
                    help="slab-decomposed matvec (SURVEY 8(e)(2), strong scaling): under torchrun one y-slab per "
                         "rank with NCCL all-to-alls; with --gpus 1, P virtual slabs on one GPU (exchange by copies)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2105_08627_b200 import svh

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    numa_cpus = bind_to_gpu_numa(local)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    case, R = workload(args.workload)
    if args.nrhs:
        R = args.nrhs
    if args.tucker is None:
        args.tucker = DEFAULT_TUCKER.get(args.workload, 0.0)
    if args.slab:
        return run_slab(args, case, R, world, rank, local)
    t0 = time.perf_counter()
    h = svh.setup_case(case, tucker_tol=args.tucker, device=local)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    # the cuFFT reference pipeline first: its full-grid spectra need the memory the matvec
    # workspace takes later
    cufft = None
    if not args.no_cufft:
        cufft = cufft_reference(h, case, R)
        torch.cuda.empty_cache()
    kz, ky, kx = h.shape
    Kt = kx * ky * kz
    stream = torch.cuda.current_stream()

    I_host = torch.from_numpy(svh_inputs.currents(h.K, R, seed=100 + rank).astype(np.complex64)).pin_memory()
    out_host = torch.empty_like(I_host).pin_memory()
    I = I_host.cuda()
    out = torch.empty_like(I)

    for _ in range(max(3, args.warmup)):
        h.matvec(I, out=out)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- device-timed region (inputs resident in HBM) ----
    h.profile(True)
    h.profile_read(reset=True)
    n0 = svh.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            h.matvec(I, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = svh.launch_count() - n0
    ms = e0.elapsed_time(e1) / args.steps
    pass_ms, pass_n = h.profile_read(reset=True)
    h.profile(False)
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = 5.0 * Kt * R * world / (ms_max / 1e3)

    # ---- end-to-end through the public API with host buffers ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # svh_matvec_host: H2D of the pinned input, the passes and D2H of the result, pipelined
    # by libsvh in RHS chunks (the copies hide behind the passes of neighbouring chunks)
    e2e_chunk = int(max(1, min(4, 4e9 // (5 * 8 * h.K))))   # RHS per pipelined slot (<= ~4 GB)
    h.matvec_host(I_host, out_host, chunk=e2e_chunk)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        h.matvec_host(I_host, out_host, chunk=e2e_chunk)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = f0.elapsed_time(f1) / args.steps
    t = torch.tensor([ms_e2e], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = 5.0 * Kt * R * world / (float(t.item()) / 1e3)
    io_bytes = I_host.numel() * 8

    # ---- roofline of the dominant kernel (live per-pass CUDA events) ----
    peaks, peak_src = load_peaks()
    # bytes and device time of each pass summed over the timed region (a step may run its RHS
    # in several workspace chunks, i.e. several launches per pass)
    # records 0-4: P5 passes A..E; record 5: whole P3s products (the auto plan picked P3s)
    if np.asarray(pass_n)[5] > 0:
        pb = np.array([sum(p3s_bytes(h, case, R))], dtype=np.float64)
        pass_ms = np.asarray(pass_ms, dtype=np.float64)[5:6]
        pass_n = np.maximum(np.asarray(pass_n)[5:6], 1)
        names = ["P3s_x_fused_yz_x"]
    else:
        pb = np.array(pass_bytes(h, R), dtype=np.float64)
        pass_ms = np.asarray(pass_ms, dtype=np.float64)[:5]
        pass_n = np.maximum(np.asarray(pass_n)[:5], 1)
        names = ["A_x_fwd", "B_y_fwd", "C_z_mac", "D_y_inv", "E_x_inv"]
    per_launch_ms = pass_ms / pass_n
    per_launch_bytes = pb * args.steps / pass_n
    dom = int(np.argmax(pass_ms))
    achieved = per_launch_bytes[dom] / (per_launch_ms[dom] / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    matvec_bytes = sum(pb)
    roof = {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": int(per_launch_bytes[dom]),
            "launches_per_step": int(pass_n[dom] // args.steps),
            "share_of_step": round(float(pass_ms[dom] / pass_ms.sum()), 4),
            "passes_ms_per_step": {n: round(float(x) / args.steps, 4) for n, x in zip(names, pass_ms)},
            "passes_frac": {n: round(float(b) / (float(x) / args.steps / 1e3) / 1e9 / float(peaks["hbm_gbs"]), 4)
                            for n, b, x in zip(names, pb, pass_ms)},
            "whole_matvec": {"bytes": int(matvec_bytes),
                             "achieved_GBs": round(matvec_bytes / (ms / 1e3) / 1e9, 1),
                             "frac": round(matvec_bytes / (ms / 1e3) / 1e9 / peak, 4)}}
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            tr = json.load(open(traffic_file)).get(case["name"], {}).get(names[dom])
            if tr:
                roof["traffic"] = tr
        except Exception:
            pass

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": {"workload": case["name"], "grid": [kx, ky, kz], "K": h.K, "nrhs_per_gpu": R,
                       "embedding": list(h.embedding), "layout": "packed [nrhs][5][K]",
                       "kernels": "tucker tol %g" % args.tucker if args.tucker else "dense octant spectra",
                       "l2": "inputs larger than L2 (working set %.1f GB/step)" % (matvec_bytes / 1e9),
                       "occupied_unknowns_per_s": 5.0 * h.K * R * world / (ms_max / 1e3),
                       "setup_s": round(t_setup, 3)},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": io_bytes,
                    "api": "svh_matvec_host (pinned host buffers, chunked H2D/compute/D2H pipeline)",
                    "host_cpus": numa_cpus},
            "gpu_launches": int(launches),
            "clocks": clk.summary()}

    if cufft is not None:
        ms_cufft, rel_cufft = cufft
        line["config"]["cufft_reference"] = {
            "ms_per_rhs": round(ms_cufft, 4), "ours_ms_per_rhs": round(ms_max / R, 4),
            "speedup_vs_cufft": round(ms_cufft / (ms_max / R), 3), "rel_l2_vs_ours": rel_cufft,
            "what": "torch.fft (cuFFT) pad+fftn, 5->5 MAC with full-grid spectra, ifftn, crop; grid layout"}

    if not args.no_plans and world == 1:
        h.close()
        torch.cuda.empty_cache()
        line["thin_grid_plans"] = thin_grid_plans(local)
    if not args.no_solve:
        line["time_to_L"] = time_to_L(args.solve_workload, local, world, rank)

    if rank == 0 and world == 1 and not args.no_cpu:
        v, dt, cores, desc = cpu_oracle_rate(case, args.cpu_budget)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    h.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
