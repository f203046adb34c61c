#!/usr/bin/env python
"""bench.py — MPKK (arXiv:1309.4349) throughput on B200.

Metric (BASELINE.json): site-updates/s of Kawasaki MC (one site update = one
attempted exchange; one sweep = N of them, R11) and HBM GB/s vs
roofline, at 1/2/4/8 GPUs.

Step (R11): one sampling interval = S=100 MPKK sweeps + one
observable sample (N_AB energy, composition, acceptance counters, cluster-size
histogram) read back to the host.

Workload (BASELINE configs[4]): a 65536 x 65536 row slab per GPU (weak
scaling, global lattice 65536 x 65536*N), omega/kT = 0.6, 50:50, random start.
The lattice (2 x 512 MiB bit-packed per GPU) is larger than L2 (126 MB), so no
flush is needed between iterations.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 runs under torchrun (one rank per GPU, NCCL halo exchange).
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "site-updates/sec (Kawasaki MC) and HBM GB/s vs roofline at 1/2/4/8 B200"
UNIT = "site-updates/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--Lx", type=int, default=65536)
    p.add_argument("--rows-per-gpu", type=int, default=0,
                   help="rows per rank (default: 65536 for --scaling weak, 65536/N for strong)")
    p.add_argument("--scaling", choices=["weak", "strong", "both"], default="both",
                   help="weak: a 65536-row slab per GPU (the headline line); strong: one 65536^2 lattice "
                        "split over the N GPUs; both (default): the weak line, and at N > 1 the strong run "
                        "attached to it as 'strong_scaling'")
    p.add_argument("--sweeps-per-step", type=int, default=100)
    p.add_argument("--omega", type=float, default=0.6)
    p.add_argument("--fraction", type=float, default=0.5)
    p.add_argument("--seed", type=int, default=20261018)
    p.add_argument("--T", type=int, default=8, help="MPKK iterations per HBM pass")
    p.add_argument("--no-ccl", action="store_true", help="skip the cluster histogram in the step")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-other-configs", action="store_true",
                   help="skip the short device-timed runs of BASELINE configs[0..3] (rank 0, N=1)")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (profiling recipe)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
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
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def other_configs(torch):
    """Short device-timed runs of the other BASELINE configs on this GPU (not
    the headline metric; context for the per-config table in DESIGN.md)."""
    from paper_1309_4349_b200 import kk
    out = []
    s = torch.cuda.current_stream()
    for name, Lx, Ly, R, om, n in [("configs[0] 64x64", 64, 64, 1, 0.5, 1000),
                                   ("configs[1] 400x400, one lattice", 400, 400, 1, 0.6, 1000),
                                   ("configs[2] 4096x4096", 4096, 4096, 1, 0.6, 100),
                                   ("configs[3] 1024 x 400x400 replicas", 400, 400, 1024, 0.6, 20)]:
        L = kk.Lattice(Lx, Ly, 0.5, om, 7, replicas=R)
        L.sweep(2, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out.append({"workload": name, "kernel": kk.plan(Lx, Ly, replicas=R, n_sm=0)["kernel"], "sweeps": n,
                    "value": n * Lx * Ly * R / (ms / 1e3), "unit": UNIT})
        L.close()
    return out


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


def kernel_counters(plan: dict):
    """Per-site-update instruction count, pipe utilisation and DRAM bytes of the
    pass kernel from the committed ncu capture of the bench lattice
    (profiles/pass_kernel_counters.json, tools/write_counters.py) — only if it
    was captured with exactly this run's launch plan (kernel, T, tile shape,
    CTA size, TMA boxes); a stale capture is refused (None, reason)."""
    try:
        with open(os.path.join(ROOT, "profiles", "pass_kernel_counters.json")) as f:
            cnt = json.load(f)
    except Exception as e:  # noqa: BLE001
        return None, f"no counters file ({e.__class__.__name__})"
    want = {k: plan[k] for k in ("kernel", "iters_per_pass", "tile_words", "tile_rows", "threads", "tma_boxes")}
    got = cnt.get("plan", {})
    if any(got.get(k) != v for k, v in want.items()):
        return None, f"counters captured for plan {got}, this run uses {want}"
    if cnt.get("source_sha256") != pass_source_sha256(plan["kernel"]):
        return None, "counters captured from different pass-kernel sources"
    return cnt, None


def pass_source_sha256(kernel: str = "planar"):
    """Fingerprint of the sources of the pass kernel the counters describe
    (the capture is refused after any change to them)."""
    import hashlib
    files = {"planar": ("kk_planar.cu", "kk_device.cuh", "kk_internal.cuh"),
             "tile": ("kk_pass.cu", "kk_device.cuh", "kk_internal.cuh")}.get(kernel, ())
    h = hashlib.sha256(kernel.encode())
    for f in files:
        with open(os.path.join(ROOT, "paper_1309_4349_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def philox_floor(upd_rate: float):
    """The R6 Philox work as a time floor: 2 Philox4x32-10 calls per 8 centres
    at the rate Philox rounds alone reach on this GPU (tools/philox_rate.cu, 4
    interleaved streams, 768-thread CTAs, one per SM; committed in
    profiles/r02_philox_rate.txt) — the pass cannot beat it whatever else it
    overlaps.  None if the measurement is not in the tree."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_philox_rate.txt")) as f:
            line = next(ln for ln in f if ln.startswith("wide") and "N=4" in ln and "threads= 768" in ln)
        calls = float(line.split(":")[1].split("G calls/s")[0]) * 1e9
    except Exception:  # noqa: BLE001
        return None
    bound = calls * 4.0
    return {"calls_per_update": 1.0 / 4.0, "philox_calls_per_s": calls, "bound_updates_per_s": bound,
            "frac": upd_rate / bound, "source": "tools/philox_rate.cu; profiles/r02_philox_rate.txt"}


# ------------------------------------------------------------------------ CPU baseline
def cpu_baseline(seconds: float, omega: float, fraction: float, seed: int):
    """The oracle as it stands (single-threaded C), on a bounded sample."""
    from oracle import oracle as O
    Lx = Ly = 1024
    lat = O.init_random(Lx, Ly, fraction, seed)
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds:
        O.run(lat, omega, seed, 1, first_sweep=n)
        n += 1
    dt = time.perf_counter() - t0
    return {"value": n * Lx * Ly / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{Lx}x{Ly} lattice, {n} MPKK sweeps, omega={omega}, single thread, "
                      f"{dt:.1f} s"}


def run_reference(a, rank, world):
    """--impl reference: the oracle on the host cores, bounded steps."""
    if rank != 0:
        return
    from oracle import oracle as O
    Lx = Ly = 1024
    lat = O.init_random(Lx, Ly, a.fraction, a.seed)
    per_step_sweeps = 2
    for w in range(a.warmup):
        O.run(lat, a.omega, a.seed, per_step_sweeps, first_sweep=w * per_step_sweeps)
    t0 = time.perf_counter()
    for k in range(a.steps):
        O.run(lat, a.omega, a.seed, per_step_sweeps, first_sweep=(a.warmup + k) * per_step_sweeps)
        O.n_ab(lat)
        O.composition(lat)
        O.cluster_histogram(lat, 1)
    dt = time.perf_counter() - t0
    v = a.steps * per_step_sweeps * Lx * Ly / dt
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u1",
        "data": "synthetic",
        "config": {"workload": f"oracle sample of configs[4]: {Lx}x{Ly}, {per_step_sweeps} sweeps + "
                               "observables per step", "omega_kT": a.omega, "fraction_A": a.fraction},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{Lx}x{Ly}, {per_step_sweeps} sweeps/step, single thread"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------ ours
def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world if world > 1 else 1)
        return
    import torch
    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    # KK_BENCH_BACKEND=gloo + KK_BENCH_DEVICE=0: functional runs of the N>1
    # path with several ranks on one GPU (NCCL refuses that); never for numbers
    backend = os.environ.get("KK_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("KK_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_1309_4349_b200 import build as B
    if rank == 0:
        B.build()
    if dist:
        dist.barrier()
    from paper_1309_4349_b200 import kk
    from paper_1309_4349_b200 import distributed as D

    ctx = dict(a=a, torch=torch, dist=dist, backend=backend, kk=kk, D=D, rank=rank, world=world, local=local)
    if a.scaling == "strong":
        rows = a.rows_per_gpu or max(4, 65536 // world)
        out = measure(ctx, rows, "strong", with_e2e=not a.no_e2e)
    else:
        out = measure(ctx, a.rows_per_gpu or 65536, "weak", with_e2e=not a.no_e2e)
        if a.scaling == "both" and world > 1:
            strong = measure(ctx, max(4, 65536 // world), "strong", with_e2e=False)
            if out is not None:
                out["strong_scaling"] = {k: strong[k] for k in ("value", "unit", "ms_per_step", "config",
                                                                 "roofline", "gpu_launches", "clocks")}
    if rank == 0:
        if world == 1 and not a.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(a.cpu_seconds, a.omega, a.fraction, a.seed)
        if world == 1 and not a.no_other_configs:
            out["other_configs"] = other_configs(torch)
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def measure(ctx, rows, scaling, with_e2e=True):
    """One bench configuration: `rows` rows per rank of a Lx x (rows * N)
    torus; W warm-up steps, K timed steps (CUDA events, max over ranks), the
    pass kernel's roofline from per-launch events, and the end-to-end run
    through the C ABI's host I/O.  Returns the JSON dict on rank 0."""
    a, torch, dist, backend, kk, D = ctx["a"], ctx["torch"], ctx["dist"], ctx["backend"], ctx["kk"], ctx["D"]
    rank, world, local = ctx["rank"], ctx["world"], ctx["local"]
    Lx, Ly = a.Lx, rows * world
    stream = torch.cuda.current_stream()
    sim = D.make_simulation(Lx, Ly, a.fraction, a.omega, a.seed, T=a.T, world=world, rank=rank,
                            device=local, stream=stream)
    N_local = Lx * rows
    passes_per_sweep = 16 // a.T

    pass_events = []

    def one_step(record):
        for _ in range(a.sweeps_per_step):
            for _p in range(passes_per_sweep):
                if record:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    sim.run_pass()
                    e1.record(stream)
                    pass_events.append((e0, e1))
                else:
                    sim.run_pass()
        return sim.observe(ccl=not a.no_ccl)

    for _ in range(a.warmup):
        one_step(False)
    torch.cuda.synchronize()
    launches0 = kk.launch_count()
    hbm_peak, sm_max_mhz, peak_src = measured_peaks()
    peak_src_hbm = peak_src
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(a.steps):
            obs = one_step(True)
        t1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = kk.launch_count() - launches0
    ms = t0.elapsed_time(t1)
    pass_ms = [e0.elapsed_time(e1) for e0, e1 in pass_events]
    if dist:
        t = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / a.steps
    updates_per_step = a.sweeps_per_step * Lx * Ly  # all ranks
    value = updates_per_step * a.steps / (ms / 1e3)

    # ---- roofline of the dominant kernel (the pass kernel), from live event timings
    pass_avg_s = float(np.mean(pass_ms)) / 1e3
    upd_per_launch = N_local * a.T / 16
    hbm_bytes_per_launch = 2 * N_local / 8  # read + write every site bit once (algorithmic)
    hbm_achieved = hbm_bytes_per_launch / pass_avg_s / 1e9
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    plan = kk.plan(Lx, Ly, y_begin=rank * rows, y_count=rows, iters_per_pass=a.T, n_sm=n_sm)
    kname = {"planar": "planar_pass_kernel", "tile": "pass_kernel"}.get(plan["kernel"], plan["kernel"])
    cnt, why = kernel_counters(plan)
    # issue peak: n_SM x 4 SMSPs x 32 lanes x 1 warp-instruction / clk at the max SM clock
    alu_peak = n_sm * 128 * sm_max_mhz * 1e6 / 1e12
    peak_src = f"{n_sm} SMs x 128 lanes x {sm_max_mhz:.0f} MHz (max SM clock, {peak_src})"
    upd_rate = upd_per_launch / pass_avg_s
    # implementation-independent floor: the Philox work R6
    # fixes (2 Philox4x32-10 calls per 8 centres, 10 rounds x 2 wide
    # multiplies + 2 three-way XORs = 40 integer ops a call: 10 ops / update,
    # plus the one multiply that splits each centre's word into d and u: 11)
    floor = 11.0
    roof = {"bound": "alu", "unit": "Tlane-op/s", "peak": alu_peak, "peak_source": peak_src,
            "kernel": kname, "plan": {k: plan[k] for k in ("kernel", "tile_words", "tile_rows", "threads",
                                                          "tma_boxes", "ctas")},
            "launch_ms": pass_avg_s * 1e3, "updates_per_launch": upd_per_launch,
            "ops_floor_per_update": floor, "floor_frac": floor * upd_rate / 1e12 / alu_peak}
    if cnt:
        lane_ops = cnt["thread_inst_per_update"] * upd_per_launch
        achieved = lane_ops / pass_avg_s / 1e12
        traffic = cnt.get("dram_bytes_per_update")
        roof.update({"achieved": achieved, "frac": achieved / alu_peak,
                     "traffic": traffic * upd_per_launch if traffic is not None else None,
                     "per_launch_ops": lane_ops, "thread_inst_per_update": cnt["thread_inst_per_update"],
                     "alu_pipe_frac": cnt.get("alu_pipe_pct", 0) / 100.0,
                     "fma_pipe_frac": cnt.get("fma_pipe_pct", 0) / 100.0,
                     "fmaheavy_pipe_frac": cnt.get("fmaheavy_pipe_pct", 0) / 100.0,
                     "issue_active_frac": cnt.get("issue_active_pct", 0) / 100.0,
                     "ops_source": cnt.get("source")})
    else:
        roof.update({"achieved": None, "frac": None, "traffic": None, "note": why})
    roof["philox_floor"] = philox_floor(upd_rate)
    roof["share_of_step"] = float(np.sum(pass_ms)) / (ms / 1.0) if ms > 0 else None
    roof["hbm"] = {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                   "frac": hbm_achieved / hbm_peak, "bytes_per_launch": hbm_bytes_per_launch,
                   "peak_source": peak_src_hbm}

    # ---- end to end through the public API: H2D of the step's lattice from pinned
    # host memory, the step, D2H of the observables (and of the lattice)
    e2e = None
    if with_e2e:
        # Every step, through the library's double-buffered host I/O (C ABI,
        # include/kk.h): upload of the step's input lattice from pinned host
        # memory (kk_upload_packed_async on a copy stream, overlapping the
        # previous step; kk_commit_upload on the compute stream), the step,
        # and the download of its result (kk_snapshot + kk_download_packed_async,
        # overlapping the next step; the last one inside the timed region).
        words = sim.packed_words()
        host_in = torch.empty(words, dtype=torch.int32, pin_memory=True)
        host_out = torch.empty(words, dtype=torch.int32, pin_memory=True)
        sim.snapshot(stream)
        cp = torch.cuda.Stream()
        sim.download_async(host_in.data_ptr(), cp)      # the current state is the first input
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        w0 = time.perf_counter()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        cp.wait_stream(stream)
        sim.upload_async(host_in.data_ptr(), cp)
        for k in range(a.steps):
            sim.commit_upload(stream)
            if k + 1 < a.steps:
                sim.upload_async(host_in.data_ptr(), cp)
            one_step(False)
            sim.snapshot(stream)
            sim.download_async(host_out.data_ptr(), cp)
        stream.wait_stream(cp)
        s1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        e_ms = max(s0.elapsed_time(s1), wall * 1e3)
        if dist:
            t = torch.tensor([e_ms], device="cuda" if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        nbytes = words * 4
        e2e = {"value": updates_per_step * a.steps / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world + 8 * 8,
               "path": "kk_upload_packed_async / kk_commit_upload / kk_snapshot / kk_download_packed_async "
                       "(C ABI) + the observables read back every step",
               "note": "per step: pinned-host->HBM upload of the step's input lattice (copy stream, overlapped "
                       "with the previous step), S sweeps + observables, lattice download (overlapped with "
                       "the next step); the last download is inside the timed region"}

    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "u1", "data": "synthetic",
            "config": {"workload": f"configs[4]: {Lx}x{rows} slab per GPU (global {Lx}x{Ly}, {scaling} scaling), "
                                   f"{a.sweeps_per_step} sweeps + observables"
                                   + ("" if a.no_ccl else " + cluster histogram") + " per step",
                       "omega_kT": a.omega, "fraction_A": a.fraction, "start": "random",
                       "iters_per_pass": a.T, "parallelism": f"slab{world}",
                       "l2": (f"inputs larger than L2 (2 x {Lx * rows // 8 // 2**20} MiB bit-packed per GPU)"
                              if Lx * rows // 8 > 126 * 2**20 else
                              f"lattice ({Lx * rows // 8 // 2**20} MiB per buffer) fits in L2: small-case run, "
                              "not a bench configuration")},
            "roofline": roof,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "observables": obs,
        }
    sim.close()
    torch.cuda.synchronize()
    return out


if __name__ == "__main__":
    main()
