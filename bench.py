"""bench.py — vehicle-steps/s of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (N=1): SURVEY §8(d) C4, the city-like synthetic network (G = 72
perturbed grid, ~133k lanes, 5,184 signalised junctions) with 2,000,000
vehicles on the network, seeded.  A step is one call of sim_step(1): the
signal kernel + the fused step kernel over all road tiles.  Each timed step is
preceded (outside its events) by an L2 flush (a 512 MiB device write), so
every step streams its state from HBM.  Device time: CUDA events on the
simulation stream.  value = sum over the timed steps of vehicles moved / time.

--impl reference times the fp64 CPU oracle (oracle/, the reference arm of
this task) on the same workload on the host's cores.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "vehicle-steps/sec"
UNIT = "vehicle-steps/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_TRAFFIC = os.path.join(ROOT, "profiles", "ncu_kstep_traffic.json")


# algorithmic bytes per vehicle-step at C4 (hot record read 24 +
# written 24, lane summaries ~2.5, events ~1-2) — the roofline's unit figure
B_ALG = 52.0


def algorithmic_bytes(n_veh, n_movers, n_lanes):
    """This implementation's own byte model of a step, reported
    beside the SURVEY figure: the 32 B vehicle record read + written per
    vehicle, per mover one more record (inbox write + read), and per lane 48 B
    (descriptor / staging + summary write, clear, read)."""
    return 64.0 * n_veh + 32.0 * n_movers + 48.0 * n_lanes


def host_cpu():
    """(cores available to this process, CPU model)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return len(os.sched_getaffinity(0)), model


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML while the timed region runs."""
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device=0):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    getattr(self.nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
                r = fn(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def make_workload(world=1, policy="fixed", scale=1.0):
    """C4 at N=1; weak scaling for N > 1: the same city recipe grown to N times
    the area (G = 72 * sqrt(N)) with 2M vehicles per GPU, spatially partitioned
    over the N GPUs with boundary migration.
    policy "maxpressure": every signalised junction runs MAX_PRESSURE (NEXT-1)."""
    import synth
    G = int(round(72 * np.sqrt(world * scale)))
    scen = synth.city(G=G, n_vehicles=int(round(2_000_000 * world * scale)), seed=4)
    if policy == "maxpressure":
        jp = scen.graph["junc_policy"]
        scen.graph["junc_policy"] = np.where(jp == synth.POLICY_FIXED, synth.POLICY_MAXP, jp).astype(np.uint8)
    return scen


def workload_config(scen, extra=None, policy="fixed", preroll=0):
    G = int(np.sqrt(len(scen.graph["junc_lane_offsets"]) - 1))
    sig = "fixed-time signals" if policy == "fixed" else "max-pressure signals (period 30 s)"
    cfg = {"workload": f"C4 city-like synthetic network (SURVEY 8(d)): G={G} perturbed grid, "
                       f"{scen.n_trips / 1e6:.3g}M vehicles on the network at t=0, {sig}; "
                       f"timed after a {preroll}-step untimed pre-roll from the t=0 placement "
                       f"(vehicles at rest) plus the warm-up steps",
           "preroll_steps": int(preroll),
           "n_vehicles": int(scen.n_trips), "n_lanes": int(scen.n_lanes),
           "n_junctions": int(len(scen.graph["junc_lane_offsets"]) - 1),
           "n_roads": int(len(scen.graph["road_lane_offsets"]) - 1),
           "l2": "flushed (512 MiB write) before every timed step",
           "seed": int(scen.params["seed"])}
    if extra:
        cfg.update(extra)
    return cfg


def cpu_baseline(scen, budget_s=20.0, max_steps=10):
    """The oracle as it stands, single-threaded, on a bounded sample (the
    first steps of the same workload from the same initial state)."""
    import oracle
    oracle.build()
    o = oracle.Oracle(scen)
    done, veh, t0 = 0, 0, time.perf_counter()
    while done < max_steps and (time.perf_counter() - t0) < budget_s:
        before = o.metrics()["vehicle_steps"]
        o.step(1)
        veh += o.metrics()["vehicle_steps"] - before
        done += 1
    dt = time.perf_counter() - t0
    ncores, model = host_cpu()
    return {"value": veh / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "host_cores": ncores, "cpu_model": model,
            "sample": f"first {done} steps of the same C4 workload ({veh} vehicle-steps, "
                      f"{dt:.1f} s, serial fp64 C++ oracle, one thread)"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    scen = make_workload(1, args.policy, args.scale)
    import oracle
    oracle.build()
    o = oracle.Oracle(scen)
    for _ in range(args.warmup):
        o.step(1)
    budget = 150.0
    done, veh, t0 = 0, 0, time.perf_counter()
    while done < args.steps and (time.perf_counter() - t0) < budget:
        before = o.metrics()["vehicle_steps"]
        o.step(1)
        veh += o.metrics()["vehicle_steps"] - before
        done += 1
    dt = time.perf_counter() - t0
    value = veh / dt
    sample = (f"{done} of {args.steps} timed steps (after {args.warmup} warm-up; the "
              f"{args.preroll}-step pre-roll of the GPU arm is skipped: minutes of serial oracle "
              f"time) of the C4 workload, {veh} vehicle-steps in {dt:.1f} s, one thread")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": done, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / max(done, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(scen, policy=args.policy, preroll=args.preroll),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "host_cores": host_cpu()[0], "cpu_model": host_cpu()[1],
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _same_device():
    # BENCH_SAME_DEVICE=1: every rank on cuda:0 with a gloo process group, to
    # exercise the multi-process path on a one-GPU box (numbers not meaningful)
    return os.environ.get("BENCH_SAME_DEVICE") == "1"


def _device_of(local_rank):
    return 0 if _same_device() else local_rank


def _max_over_ranks(x, dev):
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device="cpu" if _same_device() else dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_gpu(args, rank, world, local_rank):
    import torch
    import paper_2406_10661_b200 as p
    local_rank = _device_of(local_rank)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if rank == 0:
        p.build()
    if world > 1:
        torch.distributed.barrier()
    # weak (default): C4 per GPU, the city grown N x; strong (BASELINE configs[3],
    # "1 GPU vs 8 GPUs partitioned"): the one C4 instance split over the N GPUs
    scen = make_workload(1 if args.scaling == "strong" else world, args.policy, args.scale)
    stream = torch.cuda.Stream(dev)          # the simulation stream (events recorded on it)
    torch.cuda.set_stream(stream)
    sim = None
    if world > 1 and args.transport == "direct":
        # NEXT-2: k_step stores boundary movers straight into the
        # owner GPU's inbox over NVLink peer memory (CUDA IPC), one device
        # barrier per step; the handles are all-gathered once here.  If any
        # rank cannot map its peers, every rank falls back to NCCL p2p.
        import synth
        from paper_2406_10661_b200.sim import connect_process_group
        ok = 1
        try:
            try:
                sim = p.Sim.from_scenario(scen, device=local_rank, stream=stream.cuda_stream,
                                          world=world, rank=rank, direct=True,
                                          road_owner=synth.rcb_partition(scen, world))
            finally:
                connect_process_group(sim, world)
        except p.SimError as e:
            print(f"rank {rank}: direct transport unavailable ({e}); falling back to NCCL",
                  file=sys.stderr, flush=True)
            ok = 0
        if _max_over_ranks(1 - ok, dev) > 0:
            sim = None
            args.transport = "nccl"
    if sim is not None:
        pass
    elif world > 1:
        import synth
        nid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            nid.copy_(torch.frombuffer(bytearray(p.get_nccl_unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(nid, 0)
        sim = p.Sim.from_scenario(scen, device=local_rank, stream=stream.cuda_stream, world=world,
                                  rank=rank, nccl_id=bytes(nid.cpu().numpy()),
                                  road_owner=synth.rcb_partition(scen, world))
    else:
        sim = p.Sim.from_scenario(scen, device=local_rank, stream=stream.cuda_stream)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    sim.step(args.preroll)                               # steady state: the t=0 placement is at rest
    for _ in range(args.warmup):
        sim.step(1)
    m0 = sim.read_metrics()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sim.enable_timing(True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.fill_(k & 0xff)                      # L2 flush, outside the events
            evs[k][0].record(stream)
            sim.step(1)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = sum(a.elapsed_time(b) for a, b in evs)
    kstep_ms, ksig_ms, launches = sim.read_timing()
    sim.enable_timing(False)
    m1 = sim.read_metrics()                  # global (allreduced over ranks when partitioned)
    tot_vsteps = m1["vehicle_steps"] - m0["vehicle_steps"]
    movers = (m1["n_lane_changes"] - m0["n_lane_changes"]) + (m1["n_handoffs"] - m0["n_handoffs"]) \
        + (m1["n_finished"] - m0["n_finished"])
    t_max = _max_over_ranks(step_ms, dev) if world > 1 else step_ms
    value = tot_vsteps / (t_max / 1e3)
    # roofline of the dominant kernel (k_step), per GPU
    peak, peak_kind = peaks()
    veh_per_launch = tot_vsteps / args.steps / world         # per GPU
    survey_bytes = B_ALG * veh_per_launch                    # SURVEY 8(d) unit figure x units
    model_bytes = algorithmic_bytes(veh_per_launch, movers / args.steps / world, scen.n_lanes / world)
    kstep_avg_s = kstep_ms / 1e3 / args.steps
    achieved = survey_bytes / kstep_avg_s / 1e9
    traffic = issue = None
    if world == 1:                                        # the ncu capture of this very instance
        for path in (NCU_TRAFFIC, NCU_TRAFFIC.replace(".json", "_8m.json")):
            try:
                with open(path) as f:
                    tr = json.load(f)
                if tr.get("workload") == "C4" and tr.get("n_vehicles") == scen.n_trips:
                    traffic = tr.get("dram_bytes_per_launch")
                    issue = tr.get("issue_frac")
            except Exception:
                pass
    # e2e: RL-style loop through the public API with host buffers
    nj = len(scen.graph["junc_lane_offsets"]) - 1
    jids = np.arange(nj, dtype=np.int32)
    offs = scen.graph["junc_offset_steps"].astype(np.int64)
    e2e_steps = max(10, min(4 * args.steps, 200))          # >= 200 steps at the default: host jitter
    lane_bytes = 8 * scen.n_lanes
    host_ctl = args.policy == "fixed"                     # max pressure runs on the device
    # host fixed-time controller (C = 102 s: NS 30+3, NS-left 15+3, EW 30+3,
    # EW-left 15+3, per-junction offsets): the plan is periodic, so the phase
    # vector of every cycle second is tabulated once
    tau_phase = np.where(np.arange(102) < 33, 0, np.where(np.arange(102) < 51, 1,
                         np.where(np.arange(102) < 84, 2, 3))).astype(np.int32)
    plan = np.ascontiguousarray(tau_phase[(np.arange(102)[:, None] + offs[None, :]) % 102])
    # observation buffers: page-locked, reused every step (filled by DMA)
    obs_buf = {k: torch.empty(scen.n_lanes, dtype=torch.int32, pin_memory=True).numpy()
               for k in ("lane_count", "lane_waiting_at_end")}
    torch.cuda.synchronize()
    me0 = sim.read_metrics()
    t0 = time.perf_counter()                              # one-time setup above is outside
    for k in range(e2e_steps):
        if host_ctl:
            ph = plan[(me0["t"] + k) % 102]               # host fixed-time controller
            sim.set_signal_phase_batch(jids, ph)          # H2D: the step's control input
        sim.step(1)
        obs = sim.read_metrics(lane_stats=True, out=obs_buf)  # D2H: counters + lane queues
    e2e_dt = time.perf_counter() - t0
    e2e_v = obs["vehicle_steps"] - me0["vehicle_steps"]       # global
    e2e_val = e2e_v / e2e_dt
    if world > 1:
        e2e_val = e2e_v / _max_over_ranks(e2e_dt, dev)
    if rank != 0:
        return
    cpu = cpu_baseline(scen) if world == 1 and not args.no_cpu else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(scen, policy=args.policy, preroll=args.preroll, extra={
            "parallelism": "single GPU" if world == 1 else
            f"spatial partition over {world} GPUs (recursive coordinate bisection of road tiles), " +
            ("boundary movers stored by k_step into the owner GPU's inbox over NVLink peer memory "
             "(CUDA IPC), one device barrier per step" if args.transport == "direct" else
             "boundary-vehicle migration + lane-summary halo per step via NCCL p2p") +
            (" [all ranks on one GPU: path check, not a scaling number]" if _same_device() else ""),
            "fp64_guard_hits_per_step": (m1["n_guard_hits"] - m0["n_guard_hits"]) / args.steps}),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "k_prep + k_step_w (the step kernels, one CUDA-event window)",
                     "kernel_ms_avg": kstep_ms / args.steps,
                     "signal_kernel_ms_avg": ksig_ms / args.steps,
                     "alg_bytes_per_launch": survey_bytes,
                     "alg_bytes_per_vehicle_step": B_ALG,
                     # this implementation's own byte model (32 B records etc.)
                     "model_bytes_per_launch": model_bytes,
                     "frac_model": model_bytes / kstep_avg_s / 1e9 / peak,
                     # what the kernel actually moved (ncu dram bytes of the same instance)
                     "ncu_dram_gbs": (traffic / kstep_avg_s / 1e9) if traffic else None,
                     "ncu_dram_over_alg": (traffic / survey_bytes) if traffic else None,
                     # k_step is latency / issue bound: warp instructions
                     # issued / (148 SMs x 4 schedulers x 1965 MHz), from the ncu capture
                     "issue_frac_ncu": issue},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8 * nj if host_ctl else 0,
                "d2h_bytes_per_step": lane_bytes + 8 * 15, "steps": e2e_steps},
        "gpu_launches": int(launches),
        # ranks in the NCCL communicator / processes whose buffers are mapped (direct)
        "comm": {"transport": args.transport if world > 1 else None, "ranks": world},
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--preroll", type=int, default=200,
                    help="untimed steps before the warm-up (steady state; the t=0 placement is at rest)")
    ap.add_argument("--policy", default="fixed", choices=["fixed", "maxpressure"])
    ap.add_argument("--transport", default="nccl", choices=["direct", "nccl"],
                    help="N > 1: boundary migration + halo by NCCL p2p (north_star), or direct "
                         "peer-memory stores from k_step over CUDA IPC (NEXT-2)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: C4 per GPU (weak) or one C4 split over the N GPUs (strong)")
    ap.add_argument("--scale", type=float, default=1.0,
                    help="per-GPU size relative to C4 (4 = the 8M-vehicle single-GPU instance of SURVEY 8(d))")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(_device_of(local_rank))
        torch.distributed.init_process_group("gloo" if _same_device() else "nccl")
    run_gpu(args, rank, world, local_rank)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
