"""Benchmark of the B200 ls1-mardyn hot path (BASELINE.json metric: million
molecule-updates per second (MMUPS) and % of the FP32 roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl mardyn|reference]

One step = one pass of the whole hot path: forces and
torques at t_k on the linked-cell grid, observables, leapfrog (+ rotation),
cell rebuild by counting sort.  Default workload: BASELINE configs[1]
(1,048,576 LJTS particles, FCC 64^3, rho = 0.75, T = 0.95, rc = 2.5).
Inputs are resident in HBM when the timed region starts; L2 (126 MB) is
flushed between timed steps by writing a 256 MB buffer.  Each step is timed
with CUDA events on the context's stream; the force kernel is timed with
event nodes inside the captured step graph.

--impl reference times the fp64 CPU oracle (oracle/) as it stands on the
host cores: each step is a bounded sample of the same workload (full-shell
forces on a fixed sample of molecules), see DESIGN.md §7.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FLOP_COM_TEST = 8      # per half-shell candidate (SURVEY §8(d) flop model)
FLOP_LJ_PAIR = 20      # per in-range unique pair (incl. U, W)
FLOP_SITE_DIST = 8     # site-site separation of a rigid pair's site pair
# site-pair kernels (incl. U, W; FMA = 2): LJ 20, q-q RF 23, Q-Q ~110;
# the other polar kinds by the same closed-form count (model values)
FLOP_SITE = {("lj", "lj"): 20, ("q", "q"): 23, ("Q", "Q"): 110, ("q", "mu"): 40, ("q", "Q"): 50,
             ("mu", "mu"): 60, ("mu", "Q"): 90}
REF_SAMPLE = 32768     # molecules per --impl reference step


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)     # BASELINE configs[1]: 100 steps NVE
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="c1")
    p.add_argument("--impl", default="mardyn", choices=["mardyn", "reference"])
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    # N > 1: steps between k-d re-partitions from the measured cell loads;
    # default: 100 for the heterogeneous slab c4 (BASELINE configs[4]), else static
    p.add_argument("--rebalance-interval", type=int, default=None)
    return p.parse_args()


def pair_flops(system):
    """Algorithmic flops per in-range unique molecule pair (single component):
    every site pair of the pair (reading A1) = site separation + site kernel."""
    c = system["components"][0]
    n = {"lj": len(c["lj"]), "q": len(c["charges"]), "mu": len(c["dipoles"]), "Q": len(c["quadrupoles"])}
    if n["lj"] == 1 and n["q"] + n["mu"] + n["Q"] == 0 and len(system["components"]) == 1:
        return FLOP_LJ_PAIR                      # single-site LJ: the COM separation is the site one
    tot = 0
    for (ka, kb), f in FLOP_SITE.items():
        m = n[ka] * n[kb] * (1 if ka == kb else 2)
        tot += m * (FLOP_SITE_DIST + f)
    return tot


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def fp32_peak_tflops(num_sms, mhz):
    """FP32 CUDA-core peak: SMs x 128 lanes x 2 flops (FFMA) x clock."""
    return num_sms * 128 * 2 * mhz * 1e6 / 1e12


class Clocks:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line): an NVML thread polling every 5 ms (the timed
    region of a step is well under a millisecond), nvidia-smi as the fallback."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples, self.reasons, self.smax = [], set(), 0.0
        self.thread = None
        self.stop_flag = False
        self.p = None
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(device)).split(",")[device]) \
                if os.environ.get("CUDA_VISIBLE_DEVICES", "").replace(",", "").isdigit() else device
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def _poll(self):
        nv = self.nv
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self.stop_flag:
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, b in bits.items():
                    if r & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.nv is not None:
            import threading
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag = True
            self.thread.join()
            if not self.samples:
                return None
            return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.smax,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml, 5 ms"}
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = max(smax, float(r[2]))
                for nm, val in zip(names, r[5:9]):
                    if val.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi, 200 ms"}


def run_reference(args, system, rank, world):
    """The oracle as it stands, on the host cores (bounded sample per step)."""
    if rank != 0:
        return
    import oracle
    o = oracle.System(system)
    u = o.quantize(system["r"])
    N = len(u)
    rng = np.random.default_rng(1)
    sample = np.sort(rng.choice(N, size=min(REF_SAMPLE, N), replace=False)).astype(np.int64)
    cores = os.cpu_count()
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        o.forces(system["comp"], u, system["q"], mode="full", idx=sample, nthreads=cores)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = len(sample) * len(times) / tot / 1e6
    line = {
        "impl": "reference", "metric": "MMUPS (million molecule-updates/s)", "value": value,
        "unit": "MMUPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, BASELINE configs)",
        "config": {"workload": system["name"], "n_molecules": N, "sample_per_step": len(sample)},
        "cpu_baseline": {"value": value, "unit": "MMUPS", "cores": cores, "kind": "oracle",
                         "sample": f"full-shell fp64 forces on {len(sample)} fixed random molecules of "
                                   f"{system['name']} per step (cell lists over all {N})"},
        "e2e": {"value": value, "unit": "MMUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(system, seconds=12.0):
    """Oracle timed on the host cores on a bounded sample of the workload: all cores
    (OpenMP over molecules) and, one thread."""
    import oracle
    o = oracle.System(system)
    u = o.quantize(system["r"])
    N = len(u)
    rng = np.random.default_rng(2)
    m = min(REF_SAMPLE, N)
    sample = np.sort(rng.choice(N, size=m, replace=False)).astype(np.int64)
    cores = os.cpu_count()

    def timed(nthreads, budget, sel):
        done, t_tot, reps = 0, 0.0, 0
        while t_tot < budget and reps < 400:
            t0 = time.perf_counter()
            o.forces(system["comp"], u, system["q"], mode="full", idx=sel, nthreads=nthreads)
            t_tot += time.perf_counter() - t0
            done += len(sel)
            reps += 1
        return done / t_tot / 1e6, reps, t_tot

    value, reps, t_tot = timed(cores, seconds, sample)
    one = sample[: max(256, m // 16)]
    v1, reps1, t1 = timed(1, seconds / 3, one)
    return {"value": value, "unit": "MMUPS", "cores": cores, "kind": "oracle",
            "sample": f"{reps} x full-shell fp64 force evaluations of {m} fixed random molecules of "
                      f"{system['name']} ({t_tot:.1f} s, OpenMP over molecules)",
            "single_thread": {"value": v1, "unit": "MMUPS", "cores": 1,
                              "sample": f"{reps1} x the first {len(one)} of those molecules, one thread ({t1:.1f} s)"}}


def measure_e2e(args, system, ctx, run, world, dist, flush):
    import torch
    N = len(system["r"])
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    h_r, h_v = pin(system["r"]), pin(system["v"])
    h_c, h_id = pin(system["comp"]), pin(system["id"])
    rigid = ctx.get_grid()["kernel"] != 0
    h_q = pin(system["q"]) if rigid else None
    h_j = pin(system["j"]) if rigid else None
    out = {"r": torch.empty((N, 3), dtype=torch.float64).pin_memory(),
           "v": torch.empty((N, 3), dtype=torch.float64).pin_memory()}
    if rigid:
        out["q"] = torch.empty((N, 4), dtype=torch.float64).pin_memory()
        out["j"] = torch.empty((N, 3), dtype=torch.float64).pin_memory()
    stepper = run.step if run is not None else ctx.step
    e_ms = []
    for k in range(args.e2e_steps + 1):
        flush.zero_()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        ctx.set_molecules(h_r, h_v, comp=h_c, q=h_q, j=h_j, id=h_id, half_step=1)
        stepper(1)
        ctx.get_observables()
        ctx.get_molecules(out)
        dt = time.perf_counter() - t0
        if k > 0:
            e_ms.append(dt * 1e3)
    ms = float(np.mean(e_ms))
    if dist:
        t = torch.tensor([ms], device="cpu" if dist.get_backend() == "gloo" else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    h2d = N * (3 * 8 + 3 * 8 + 4 + 8 + (7 * 8 if rigid else 0))
    d2h = N * (3 * 8 + 3 * 8 + (7 * 8 if rigid else 0)) + 64
    return {"value": N / (ms / 1e3) / 1e6, "unit": "MMUPS", "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "what": "set_molecules(pinned host) + step(1) + get_observables + get_molecules(pinned host)"
                    + (" on every rank (global arrays in, owned molecules out), max over ranks" if world > 1 else "")}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import scenarios as S
    system = S.config(args.config)
    if args.impl == "reference":
        return run_reference(args, system, rank, world)

    import torch
    # MARDYN_BENCH_ONE_DEVICE=1 (tests only, never the driver): every rank on cuda:0 with a
    # gloo process group, the library's transport through MARDYN_NCCL_LIB (the one-GPU NCCL
    # stand-in of tests/nccl_shim.c) -- exercises this N > 1 path on a one-GPU box
    one_dev = os.environ.get("MARDYN_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        # torch.distributed launches the ranks and broadcasts the library's NCCL unique id;
        # the halo exchange, migration, rebalance and observable reductions run on the
        # library's own communicator (include/mardyn.h)
        import torch.distributed as dist
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1408_4599_b200 import build as b
    from paper_1408_4599_b200 import mardyn
    if rank == 0 or world == 1:
        b.build()
    if dist:
        dist.barrier()
    N = len(system["r"])
    stream = torch.cuda.Stream()
    rebalance = args.rebalance_interval if args.rebalance_interval is not None else (100 if args.config == "c4" else 0)
    if world > 1:
        # spatial k-d decomposition (§4) with halo exchange and
        # migration over NCCL every step; one rank per GPU
        with torch.cuda.stream(stream):
            run = mardyn.DecomposedRun(system, world, transport="nccl", rank=rank, stream=stream,
                                       rebalance_interval=rebalance)
        ctx = run.ctxs[0]
        stepper = run.step
    else:
        ctx = mardyn.from_system(system, stream=stream)
        run = None
        stepper = ctx.step
    for _ in range(args.warmup):
        stepper(1)
    ctx.get_observables()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = Clocks(local)
    step_ms, force_ms = [], []
    l0 = ctx.launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.zero_()                          # L2 flush, outside the events
            stream.synchronize()
            if dist:
                dist.barrier()
            ev[k][0].record(stream)
            stepper(1)
            ev[k][1].record(stream)
            stream.synchronize()
            force_ms.append(ctx.last_step_timing()["force_ms"])
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = ctx.launch_count() - l0
    step_ms = [a.elapsed_time(e) for a, e in ev]
    obs = run.observables() if run is not None else ctx.get_observables()
    tot_ms = float(sum(step_ms))
    if dist:
        t = torch.tensor([tot_ms], device="cpu" if dist.get_backend() == "gloo" else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        dist.barrier()
    # whole job: the N molecules of the system are updated once per step, shared among the
    # ranks of the spatial decomposition (strong scaling: N is fixed as the GPU count grows)
    value = N * args.steps / (tot_ms / 1e3) / 1e6
    # ---- roofline of the dominant kernel (force): algorithmic flops
    ncand_half = obs["n_candidates"] / 2.0
    flops = FLOP_COM_TEST * ncand_half + pair_flops(system) * obs["n_pairs"]
    f_ms = float(np.mean(force_ms)) if force_ms and min(force_ms) > 0 else None
    pk = peaks()
    props = torch.cuda.get_device_properties(local)
    peak = fp32_peak_tflops(props.multi_processor_count, pk.get("sm_max_mhz", 1965.0))
    # per GPU: the method's work of the whole system shared by the ranks, over one rank's force time
    achieved = flops / world / (f_ms / 1e3) / 1e12 if f_ms else None
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "force_traffic.json")))
        traffic = prof.get(args.config)
    except Exception:
        pass
    l1 = None                      # the force kernel's L1 / shared data-pipe utilisation (ncu, committed)
    try:
        l1 = json.load(open(os.path.join(ROOT, "profiles", "l1_pipe.json"))).get(args.config)
    except Exception:
        pass
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": {0: "k_force_lj1", 1: "k_force_rigid3"}.get(ctx.get_grid()["kernel"], "k_force_rigid"),
                "force_ms": f_ms, "force_share": (f_ms * args.steps / tot_ms) if f_ms else None,
                "algorithmic_gflop_per_launch": flops / world / 1e9,
                "flop_model": "8 x half-shell COM candidates + per unique in-range pair: sum over site pairs of "
                              "(8 separation + kernel: LJ 20, q-q RF 23, Q-Q 110) (SURVEY 8(d)); single-site LJ: 20",
                "peak_note": "FP32 CUDA cores: SMs x 128 x 2 x sm_max_mhz (MEASURED_PEAKS.json), derived",
                "l1_data_pipe_frac": l1,
                "l1_note": "fraction of the L1/shared data pipe's peak the force kernel used under ncu "
                           "(profiles/l1_pipe.json): the single-site kernel's main loop is bound by it"}
    # ---- end to end through the C ABI with pinned host buffers: every step uploads the
    #      molecules (set_molecules from pinned host arrays, exact resume) and reads back the
    #      observables and the molecules (get_molecules into pinned host arrays); at N > 1 each
    #      rank does this on its own context of the decomposed run, time = max over ranks
    e2e = None
    if args.e2e_steps > 0:
        try:
            e2e = measure_e2e(args, system, ctx, run, world, dist, flush)
        except Exception as ex:                     # the device-timed line must still print
            e2e = {"error": repr(ex)[:300]}
    if rank != 0:
        return
    cpu = None if args.no_cpu_baseline or world > 1 else cpu_baseline(system)
    line = {
        "metric": "MMUPS (million molecule-updates/s)", "value": value, "unit": "MMUPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded generator of BASELINE configs, no checkpoints)",
        "config": {"workload": system["name"], "n_molecules": N, "steps_per_run": args.steps,
                   "parallelism": (f"k-d tree spatial decomposition over {world} GPUs, halo exchange + "
                                   "migration by NCCL send/recv every step (library-owned communicator), "
                                   f"rebalance every {rebalance} steps" if rebalance else "static partition")
                                  if world > 1 else "single GPU",
                   "l2": "flushed between timed steps (256 MB write)",
                   "arithmetic": "fp32 forces (packed fp32x2), u32 fixed-point positions, fp64 sums",
                   "pair_interactions_per_s": obs["n_pairs"] * args.steps / (tot_ms / 1e3)},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clk,
        "observables": {k: obs[k] for k in ("step", "U_pot", "virial", "T", "n_pairs", "n_candidates")},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
