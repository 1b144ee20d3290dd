"""Thin ctypes binding of include/sim.h (argument marshalling only).

Every step of the simulation runs in the CUDA kernels of libsim_b200.so; this
module only converts numpy arrays / dicts to the C structs and back.  There is
no CPU fallback: if the extension is missing or no GPU is present, the calls
fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .build import LIB

SIM_OK, SIM_E_INVALID, SIM_E_RANGE, SIM_E_OOM, SIM_E_CUDA, SIM_E_NCCL, SIM_E_STATE, \
    SIM_E_CAPACITY = range(8)
STATUS_NAMES = ["SIM_OK", "SIM_E_INVALID", "SIM_E_RANGE", "SIM_E_OOM", "SIM_E_CUDA",
                "SIM_E_NCCL", "SIM_E_STATE", "SIM_E_CAPACITY"]

P = C.c_void_p


class SimError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


class sim_graph(C.Structure):
    _fields_ = [("n_lanes", C.c_int32), ("n_roads", C.c_int32), ("n_junctions", C.c_int32)] + \
        [(n, P) for n in ("lane_length", "lane_max_speed", "lane_road", "lane_junction",
                          "lane_left", "lane_right", "succ_offsets", "succ_lanes", "lane_turn",
                          "lane_kind", "tidal_partner", "lane_dir0", "road_lane_offsets",
                          "road_lanes", "junc_lane_offsets", "junc_lanes", "junc_phase_offsets",
                          "phase_green", "phase_green_steps", "junc_policy", "junc_offset_steps")]


class sim_trips(C.Structure):
    _fields_ = [("n_trips", C.c_int32)] + \
        [(n, P) for n in ("depart_step", "on_network_at_t0", "route_offsets", "route_roads",
                          "start_lane", "start_s", "start_v", "end_s", "profile")]


class sim_params(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("dt", C.c_float), ("n_profiles", C.c_int32),
                ("profiles", P), ("politeness", C.c_float), ("b_hard", C.c_float),
                ("b_safe", C.c_float), ("v_wait", C.c_float), ("queue_zone_m", C.c_float),
                ("yellow_steps", C.c_int32), ("lookahead_lanes", C.c_int32),
                ("exact_mode", C.c_int32), ("record_decisions", C.c_int32),
                ("device", C.c_int32), ("stream", P), ("rank", C.c_int32),
                ("world", C.c_int32), ("loopback", C.c_int32), ("direct", C.c_int32), ("nccl_id", P),
                ("road_owner", P), ("max_pressure_period", C.c_int32),
                ("vehicle_seed", P), ("vehicle_rng_id", P), ("road_group", P),
                ("n_groups", C.c_int32), ("barrier_timeout_ms", C.c_int32),
                ("alloc", P), ("free_", P), ("alloc_ctx", P), ("no_step_graphs", C.c_int32)]


class sim_sizes(C.Structure):
    _fields_ = [("n_vehicles", C.c_int32), ("n_lanes", C.c_int32), ("n_junctions", C.c_int32),
                ("n_tiles", C.c_int32), ("device_bytes", C.c_int64)]


class sim_state(C.Structure):
    _fields_ = [("t", C.c_int32)] + [(n, P) for n in (
        "status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time", "s", "v",
        "junc_policy", "junc_phase", "junc_elapsed", "junc_yellow_left", "junc_pending",
        "junc_remaining",
        "lane_dir", "lane_signal", "lane_offsets", "lane_order")]


class sim_decisions(C.Structure):
    _fields_ = [(n, P) for n in ("leader_vid", "leader_hops", "phantom", "old_follower_vid",
                                 "side_vid", "lc", "handoffs", "accel", "finished", "inserted",
                                 "guard")]


class sim_metrics(C.Structure):
    _fields_ = [("t", C.c_int32)] + [(n, C.c_int64) for n in (
        "n_pending", "n_driving", "n_finished", "vehicle_steps", "sum_travel_steps",
        "sum_wait_steps_finished", "sum_depart_delay", "n_lane_changes", "n_handoffs",
        "n_inserted", "n_guard_hits")] + [("att_finished", C.c_double),
                                          ("sum_time_driving", C.c_int64), ("att_all", C.c_double),
                                          ("lane_count", P), ("lane_waiting_at_end", P),
                                          ("road_avg_speed", P)]


ABI_FUNCTIONS = ["sim_create", "sim_get_nccl_unique_id", "sim_ipc_export", "sim_ipc_connect",
                 "sim_repartition", "sim_read_state_global", "sim_partition", "sim_step", "sim_sync", "sim_set_signal_phase",
                 "sim_set_signal_phase_batch", "sim_set_lane_direction",
                 "sim_set_lane_direction_batch", "sim_query_sizes", "sim_read_state",
                 "sim_read_decisions", "sim_read_metrics", "sim_read_group_metrics", "sim_set_signal_policy", "sim_set_signal_policy_batch", "sim_set_signal_duration", "sim_set_signal_duration_batch", "sim_set_vehicle_route", "sim_set_vehicle_route_batch", "sim_set_lane_max_speed", "sim_set_lane_max_speed_batch", "sim_set_lane_restriction", "sim_set_lane_restriction_batch", "sim_load_state", "sim_load_state_inbox", "sim_read_state_device",
                 "sim_enable_timing", "sim_read_timing", "sim_destroy", "sim_last_error"]

_lib = None


def load_library(path=LIB):
    """Load libsim_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"CUDA extension {path} is missing; run "
                          "`python -m paper_2406_10661_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(path)
    i32, h = C.c_int32, C.c_void_p
    sig = {
        "sim_create": [P, P, P, C.POINTER(C.c_void_p)],
        "sim_get_nccl_unique_id": [P], "sim_partition": [P, P, P, P, P],
        "sim_ipc_export": [h, P, i32, P], "sim_ipc_connect": [h, P, i32],
        "sim_repartition": [h, P, P], "sim_read_state_global": [h, P],
        "sim_step": [h, i32], "sim_sync": [h],
        "sim_set_signal_phase": [h, i32, i32], "sim_set_signal_phase_batch": [h, i32, P, P],
        "sim_set_lane_direction": [h, i32, i32], "sim_set_lane_direction_batch": [h, i32, P, P],
        "sim_query_sizes": [h, P], "sim_read_state": [h, P], "sim_read_decisions": [h, P],
        "sim_read_metrics": [h, P], "sim_read_group_metrics": [h, i32, P],
        "sim_set_signal_policy": [h, i32, i32], "sim_set_signal_policy_batch": [h, i32, P, P],
        "sim_set_signal_duration": [h, i32, i32], "sim_set_signal_duration_batch": [h, i32, P, P],
        "sim_set_vehicle_route": [h, i32, i32, P, C.c_float],
        "sim_set_vehicle_route_batch": [h, i32, P, P, P, P],
        "sim_set_lane_max_speed": [h, i32, C.c_float], "sim_set_lane_max_speed_batch": [h, i32, P, P],
        "sim_set_lane_restriction": [h, i32, i32], "sim_set_lane_restriction_batch": [h, i32, P, P],
        "sim_load_state": [h, P], "sim_load_state_inbox": [h, P, P], "sim_destroy": [h],
        "sim_read_state_device": [h, P],
        "sim_enable_timing": [h, i32], "sim_read_timing": [h, P, P, P],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int32
    lib.sim_last_error.argtypes = [h]
    lib.sim_last_error.restype = C.c_char_p
    _lib = lib
    return lib


def _ptr(a):
    return C.c_void_p(a.ctypes.data)        # (data_as is ~2x slower on the per-step path)


_GRAPH_DT = dict(lane_length=np.float32, lane_max_speed=np.float32, lane_road=np.int32,
                 lane_junction=np.int32, lane_left=np.int32, lane_right=np.int32,
                 succ_offsets=np.int32, succ_lanes=np.int32, lane_turn=np.uint8,
                 lane_kind=np.uint8, tidal_partner=np.int32, lane_dir0=np.uint8,
                 road_lane_offsets=np.int32, road_lanes=np.int32, junc_lane_offsets=np.int32,
                 junc_lanes=np.int32, junc_phase_offsets=np.int32, phase_green=np.uint8,
                 phase_green_steps=np.int32, junc_policy=np.uint8, junc_offset_steps=np.int32)
_TRIP_DT = dict(depart_step=np.int32, on_network_at_t0=np.uint8, route_offsets=np.int32,
                route_roads=np.int32, start_lane=np.int32, start_s=np.float32,
                start_v=np.float32, end_s=np.float32, profile=np.uint8)


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


def torch_allocator(device=0, stream=None):
    """(alloc, free_) callbacks of sim_params backed by PyTorch's caching
    allocator on `device` (BASELINE.json north_star: PyTorch provides the
    device memory).  Keep the returned pair alive as long as the handle."""
    import torch

    def _alloc(n, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(n), device=device, stream=stream)
        except Exception:
            return None

    def _free(p, ctx):
        torch.cuda.caching_allocator_delete(p)
    return ALLOC_FN(_alloc), FREE_FN(_free)


def _marshal(graph, trips, profiles, params, device=0, stream=None, exact_mode=False,
             record_decisions=False, world=1, rank=0, loopback=False, nccl_id=None,
             road_owner=None, direct=False, barrier_timeout_ms=0, allocator=None,
             step_graphs=True):
    g = {k: np.ascontiguousarray(graph[k], dtype=dt) for k, dt in _GRAPH_DT.items()}
    tr = {k: np.ascontiguousarray(trips[k], dtype=dt) for k, dt in _TRIP_DT.items()}
    prof = np.ascontiguousarray(profiles, dtype=np.float32).reshape(-1, 6)
    keep = [g, tr, prof]
    n_lanes = int(g["lane_length"].shape[0])
    n_j = int(g["junc_lane_offsets"].shape[0] - 1)
    n = int(tr["depart_step"].shape[0])
    G = sim_graph(n_lanes, int(g["road_lane_offsets"].shape[0] - 1), n_j,
                  *[_ptr(g[nm]) for nm, _ in sim_graph._fields_[3:]])
    T = sim_trips(n, *[_ptr(tr[nm]) for nm, _ in sim_trips._fields_[1:]])
    nid = None
    if nccl_id is not None:
        nid = np.frombuffer(bytes(nccl_id), dtype=np.uint8).copy()
        keep.append(nid)
    own = None
    if road_owner is not None:
        own = np.ascontiguousarray(road_owner, np.int32)
        keep.append(own)
    Pm = sim_params(int(params["seed"]), float(params.get("dt", 1.0)), prof.shape[0],
                    _ptr(prof), params["politeness"], params["b_hard"], params["b_safe"],
                    params["v_wait"], params["queue_zone_m"], params["yellow_steps"],
                    params["lookahead_lanes"], int(exact_mode), int(record_decisions),
                    int(device), C.c_void_p(stream) if stream else None, int(rank),
                    int(world), int(bool(loopback)), int(bool(direct)),
                    _ptr(nid) if nid is not None else None,
                    _ptr(own) if own is not None else None,
                    int(params.get("max_pressure_period", 30)),
                    *_batch_arrays(params, keep), int(barrier_timeout_ms),
                    C.cast(allocator[0], C.c_void_p) if allocator else None,
                    C.cast(allocator[1], C.c_void_p) if allocator else None, None,
                    int(not step_graphs))
    if allocator:
        keep.append(allocator)
    return G, T, Pm, keep


def _batch_arrays(params, keep):
    """Optional batched-environment inputs (sim_params.vehicle_seed,
    vehicle_rng_id, road_group, n_groups)."""
    out = []
    for name, dt in (("vehicle_seed", np.uint64), ("vehicle_rng_id", np.int32),
                     ("road_group", np.int32)):
        a = params.get(name)
        if a is None:
            out.append(None)
        else:
            a = np.ascontiguousarray(a, dt)
            keep.append(a)
            out.append(_ptr(a))
    out.append(int(params.get("n_groups", 0)))
    return out


def connect_process_group(sim, world, group=None):
    """Collective IPC connect for the direct transport; `sim` may be None on a
    rank whose sim_create failed (it still takes part, and all ranks raise)."""
    import torch.distributed as dist
    mine = None
    try:
        mine = sim.ipc_export() if sim is not None else None
    except SimError:
        pass
    blobs = [None] * world
    dist.all_gather_object(blobs, mine, group=group)
    if any(b is None for b in blobs):
        raise SimError(6, "direct transport: a rank could not create or export its buffers")
    sim.ipc_connect(blobs)


def get_nccl_unique_id():
    """128-byte NCCL unique id for a partitioned multi-process run."""
    lib = load_library()
    buf = np.zeros(128, np.uint8)
    st = lib.sim_get_nccl_unique_id(_ptr(buf))
    if st != SIM_OK:
        raise SimError(st, (lib.sim_last_error(None) or b"").decode())
    return bytes(buf)


def partition(graph, trips, profiles, params, world, road_owner=None):
    """Host-only partition + exchange-plan sizes (sim_partition; no GPU needed).

    Returns (road_owner [n_roads], mig_cap [world, world], halo [world, world])."""
    lib = load_library()
    G, T, Pm, keep = _marshal(graph, trips, profiles, params, world=world,
                              road_owner=road_owner)
    nr = G.n_roads
    own = np.zeros(nr, np.int32)
    sizes = np.zeros(world * world * 2, np.int32)
    st = lib.sim_partition(C.byref(G), C.byref(T), C.byref(Pm), _ptr(own), _ptr(sizes))
    if st != SIM_OK:
        raise SimError(st, (lib.sim_last_error(None) or b"").decode())
    sizes = sizes.reshape(world, world, 2)
    return own, sizes[:, :, 0].copy(), sizes[:, :, 1].copy()


class Sim:
    """One simulation handle (sim_create ... sim_destroy)."""

    def __init__(self, graph, trips, profiles, params, device=0, stream=None,
                 exact_mode=False, record_decisions=False, world=1, rank=0, loopback=False,
                 nccl_id=None, road_owner=None, direct=False, barrier_timeout_ms=0,
                 allocator=None, step_graphs=True):
        """allocator: None (cudaMalloc), "torch" (PyTorch's caching allocator,
        torch_allocator) or an (alloc, free_) pair of ALLOC_FN / FREE_FN.
        step_graphs: sim_step(n >= 12) replays a captured 6-step CUDA graph
        (sim_params.no_step_graphs = 0)."""
        lib = load_library()
        self.lib = lib
        if allocator == "torch":
            allocator = torch_allocator(device, stream)
        self._allocator = allocator                   # the callbacks must outlive the handle
        G, T, Pm, keep = _marshal(graph, trips, profiles, params, device, stream, exact_mode,
                                  record_decisions, world, rank, loopback, nccl_id, road_owner,
                                  direct, barrier_timeout_ms, allocator, step_graphs)
        self.n_lanes, self.n_junctions, self.n = G.n_lanes, G.n_junctions, T.n_trips
        self.n_roads = G.n_roads
        self.world, self.rank = max(1, int(world)), int(rank)
        hh = C.c_void_p()
        st = lib.sim_create(C.byref(G), C.byref(T), C.byref(Pm), C.byref(hh))
        if st != SIM_OK:
            raise SimError(st, (lib.sim_last_error(None) or b"").decode())
        self.h = hh
        self.record = bool(record_decisions)

    @classmethod
    def from_scenario(cls, scen, **kw):
        return cls(scen.graph, scen.trips, scen.profiles, scen.params, **kw)

    def _chk(self, st):
        if st != SIM_OK:
            raise SimError(st, (self.lib.sim_last_error(self.h) or b"").decode())

    def ipc_export(self):
        """This rank's CUDA IPC handles (direct transport across processes)."""
        n = C.c_int32(0)
        self._chk(self.lib.sim_ipc_export(self.h, None, 0, C.byref(n)))
        buf = np.zeros(n.value, np.uint8)
        self._chk(self.lib.sim_ipc_export(self.h, _ptr(buf), n.value, C.byref(n)))
        return bytes(buf)

    def ipc_connect(self, blobs):
        """Map the peers' buffers; blobs = every rank's ipc_export() in rank order."""
        n = len(blobs[0])
        a = np.frombuffer(b"".join(blobs), np.uint8).copy()
        self._chk(self.lib.sim_ipc_connect(self.h, _ptr(a), n))

    def connect_process_group(self, group=None):
        """All-gather the IPC handles over torch.distributed and connect.
        Collective: every rank takes part even if its export fails, and then
        every rank raises."""
        connect_process_group(self, self.world, group)

    def repartition(self, road_owner=None):
        """Hand road tiles to new owners at this step boundary (direct
        transport); road_owner None = rebalance by the current vehicle counts.
        Returns the number of tiles that moved."""
        moved = C.c_int32(0)
        own = None if road_owner is None else np.ascontiguousarray(road_owner, np.int32)
        self._chk(self.lib.sim_repartition(self.h, None if own is None else _ptr(own),
                                           C.byref(moved)))
        return moved.value

    def step(self, n=1):
        self._chk(self.lib.sim_step(self.h, int(n)))

    def sync(self):
        self._chk(self.lib.sim_sync(self.h))

    def set_signal_phase(self, junction, phase):
        self._chk(self.lib.sim_set_signal_phase(self.h, int(junction), int(phase)))

    def set_signal_phase_batch(self, junctions, phases):
        j = np.ascontiguousarray(junctions, np.int32)
        p = np.ascontiguousarray(phases, np.int32)
        self._chk(self.lib.sim_set_signal_phase_batch(self.h, len(j), _ptr(j), _ptr(p)))

    def set_lane_direction(self, lane, d):
        self._chk(self.lib.sim_set_lane_direction(self.h, int(lane), int(d)))

    def set_lane_direction_batch(self, lanes, dirs):
        l = np.ascontiguousarray(lanes, np.int32)
        d = np.ascontiguousarray(dirs, np.int32)
        self._chk(self.lib.sim_set_lane_direction_batch(self.h, len(l), _ptr(l), _ptr(d)))

    def query_sizes(self):
        s = sim_sizes()
        self._chk(self.lib.sim_query_sizes(self.h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in sim_sizes._fields_}

    def read_state(self, lane_order=False, global_view=False):
        """vid-indexed state; global_view (collective) = every partition's
        vehicles, also across processes (sim_read_state_global)."""
        n, nj, nl = self.n, self.n_junctions, self.n_lanes
        b = dict(status=np.zeros(n, np.uint8), lane=np.zeros(n, np.int32),
                 cursor=np.zeros(n, np.int32), wait_steps=np.zeros(n, np.int32),
                 insert_time=np.zeros(n, np.int32), arrive_time=np.zeros(n, np.int32),
                 s=np.zeros(n, np.float32), v=np.zeros(n, np.float32),
                 junc_policy=np.zeros(nj, np.uint8), junc_phase=np.zeros(nj, np.int32),
                 junc_elapsed=np.zeros(nj, np.int32), junc_yellow_left=np.zeros(nj, np.int32),
                 junc_pending=np.zeros(nj, np.int32), junc_remaining=np.zeros(nj, np.int32),
                 lane_dir=np.zeros(nl, np.uint8), lane_signal=np.zeros(nl, np.uint8))
        if lane_order:
            b["lane_offsets"] = np.zeros(nl + 1, np.int32)
            b["lane_order"] = np.zeros(max(n, 1), np.int32)
        st = sim_state(0, *[_ptr(b[nm]) if nm in b else None for nm, _ in sim_state._fields_[1:]])
        fn = self.lib.sim_read_state_global if global_view else self.lib.sim_read_state
        self._chk(fn(self.h, C.byref(st)))
        b["t"] = st.t
        if lane_order:
            b["lane_order"] = b["lane_order"][:b["lane_offsets"][-1]]
        return b

    def read_state_device(self, out=None):
        """The vid-indexed state into torch tensors on this handle's device
        (sim_read_state_device; stream-ordered, no synchronisation).  `out`:
        dict of preallocated tensors (reused across calls) or None."""
        import torch
        n = self.n
        dev = torch.device("cuda", torch.cuda.current_device())
        spec = dict(status=torch.uint8, lane=torch.int32, cursor=torch.int32, wait_steps=torch.int32,
                    insert_time=torch.int32, arrive_time=torch.int32, s=torch.float32, v=torch.float32)
        if out is None:
            out = {k: torch.empty(n, dtype=dt, device=dev) for k, dt in spec.items()}
            out["lane_signal"] = torch.empty(self.n_lanes, dtype=torch.uint8, device=dev)
            out["junc_phase"] = torch.empty(max(self.n_junctions, 1), dtype=torch.int32, device=dev)
        st = sim_state(0, *[C.c_void_p(out[nm].data_ptr()) if nm in out else None
                            for nm, _ in sim_state._fields_[1:]])
        self._chk(self.lib.sim_read_state_device(self.h, C.byref(st)))
        out["t"] = st.t
        return out

    def load_state(self, state, to_inbox=None):
        n, nj, nl = self.n, self.n_junctions, self.n_lanes
        conv = dict(status=np.uint8, lane=np.int32, cursor=np.int32, wait_steps=np.int32,
                    insert_time=np.int32, arrive_time=np.int32, s=np.float32, v=np.float32,
                    junc_policy=np.uint8, junc_phase=np.int32, junc_elapsed=np.int32,
                    junc_yellow_left=np.int32, junc_pending=np.int32, lane_dir=np.uint8)
        b = {k: np.ascontiguousarray(state[k], dtype=dt) for k, dt in conv.items()}
        if "junc_remaining" in state:                      # optional (NULL = no timers)
            b["junc_remaining"] = np.ascontiguousarray(state["junc_remaining"], dtype=np.int32)
        st = sim_state(int(state["t"]), *[_ptr(b[nm]) if nm in b else None
                                          for nm, _ in sim_state._fields_[1:]])
        if to_inbox is None:
            self._chk(self.lib.sim_load_state(self.h, C.byref(st)))
        else:
            ti = np.ascontiguousarray(to_inbox, np.uint8)
            assert ti.shape == (n,)
            self._chk(self.lib.sim_load_state_inbox(self.h, C.byref(st), _ptr(ti)))

    def read_decisions(self):
        n = self.n
        b = dict(leader_vid=np.zeros(n, np.int32), leader_hops=np.zeros(n, np.int8),
                 phantom=np.zeros(n, np.int8), old_follower_vid=np.zeros(n, np.int32),
                 side_vid=np.zeros(4 * n, np.int32), lc=np.zeros(n, np.int8),
                 handoffs=np.zeros(n, np.int8), accel=np.zeros(n, np.float32),
                 finished=np.zeros(n, np.int8), inserted=np.zeros(n, np.int8),
                 guard=np.zeros(n, np.uint8))
        d = sim_decisions(*[_ptr(b[nm]) for nm, _ in sim_decisions._fields_])
        self._chk(self.lib.sim_read_decisions(self.h, C.byref(d)))
        b["side_vid"] = b["side_vid"].reshape(n, 4)
        return b

    def read_metrics(self, lane_stats=False, road_speed=False, out=None):
        """Global counters (+ per-lane queue statistics / road speeds).  `out`
        (optional dict: lane_count, lane_waiting_at_end, road_avg_speed) gives
        caller-owned arrays to fill instead of fresh ones; page-locked arrays
        (e.g. torch.empty(..., pin_memory=True).numpy()) are filled by DMA."""
        m = sim_metrics()
        out = out or {}

        def buf(name, n, dt):
            a = out.get(name)
            if a is None:
                return np.zeros(n, dt)
            assert a.dtype == dt and a.shape == (n,) and a.flags.c_contiguous, name
            return a
        bufs = None
        if lane_stats:
            bufs = (buf("lane_count", self.n_lanes, np.int32),
                    buf("lane_waiting_at_end", self.n_lanes, np.int32))
            m.lane_count = _ptr(bufs[0])
            m.lane_waiting_at_end = _ptr(bufs[1])
        rs = None
        if road_speed:
            rs = buf("road_avg_speed", self.n_roads, np.float32)
            m.road_avg_speed = _ptr(rs)
        self._chk(self.lib.sim_read_metrics(self.h, C.byref(m)))
        out = {n: getattr(m, n) for n, _ in sim_metrics._fields_[:-3]}
        if bufs is not None:
            out["lane_count"], out["lane_waiting_at_end"] = bufs
        if rs is not None:
            out["road_avg_speed"] = rs
        return out

    def set_signal_policy(self, junction, policy):
        self._chk(self.lib.sim_set_signal_policy(self.h, int(junction), int(policy)))

    def set_signal_policy_batch(self, junctions, policies):
        j = np.ascontiguousarray(junctions, np.int32)
        p = np.ascontiguousarray(policies, np.int32)
        self._chk(self.lib.sim_set_signal_policy_batch(self.h, len(j), _ptr(j), _ptr(p)))

    def set_signal_duration(self, junction, steps):
        self._chk(self.lib.sim_set_signal_duration(self.h, int(junction), int(steps)))

    def set_signal_duration_batch(self, junctions, steps):
        j = np.ascontiguousarray(junctions, np.int32)
        d = np.ascontiguousarray(steps, np.int32)
        self._chk(self.lib.sim_set_signal_duration_batch(self.h, len(j), _ptr(j), _ptr(d)))

    def set_vehicle_route(self, vid, roads, end_s):
        r = np.ascontiguousarray(roads, np.int32)
        self._chk(self.lib.sim_set_vehicle_route(self.h, int(vid), len(r), _ptr(r), float(end_s)))

    def set_vehicle_route_batch(self, vids, routes, end_s):
        """routes: list of road sequences, one per vid."""
        v = np.ascontiguousarray(vids, np.int32)
        off = np.zeros(len(routes) + 1, np.int32)
        off[1:] = np.cumsum([len(r) for r in routes])
        rr = np.ascontiguousarray(np.concatenate([np.asarray(r, np.int32) for r in routes])
                                  if routes else np.zeros(0, np.int32), np.int32)
        e = np.ascontiguousarray(end_s, np.float32)
        self._chk(self.lib.sim_set_vehicle_route_batch(self.h, len(v), _ptr(v), _ptr(off), _ptr(rr), _ptr(e)))

    def set_lane_max_speed(self, lane, v):
        self._chk(self.lib.sim_set_lane_max_speed(self.h, int(lane), float(v)))

    def set_lane_max_speed_batch(self, lanes, speeds):
        l = np.ascontiguousarray(lanes, np.int32)
        v = np.ascontiguousarray(speeds, np.float32)
        self._chk(self.lib.sim_set_lane_max_speed_batch(self.h, len(l), _ptr(l), _ptr(v)))

    def set_lane_restriction(self, lane, flag):
        self._chk(self.lib.sim_set_lane_restriction(self.h, int(lane), int(flag)))

    def set_lane_restriction_batch(self, lanes, flags):
        l = np.ascontiguousarray(lanes, np.int32)
        f = np.ascontiguousarray(flags, np.int32)
        self._chk(self.lib.sim_set_lane_restriction_batch(self.h, len(l), _ptr(l), _ptr(f)))

    def read_group_metrics(self, n_groups):
        """Per-group metrics (batched environments, sim_read_group_metrics)."""
        arr = (sim_metrics * int(n_groups))()
        self._chk(self.lib.sim_read_group_metrics(self.h, int(n_groups), arr))
        return [{n: getattr(m, n) for n, _ in sim_metrics._fields_[:-3]} for m in arr]

    def enable_timing(self, on=True):
        self._chk(self.lib.sim_enable_timing(self.h, int(on)))

    def read_timing(self):
        """(step-kernel ms, signal-kernel ms, kernel launches) of the timing window."""
        a, b, n = C.c_double(), C.c_double(), C.c_int64()
        self._chk(self.lib.sim_read_timing(self.h, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value

    def destroy(self):
        if getattr(self, "h", None):
            self.lib.sim_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def sim_create(graph, trips, profiles, params, **kw):
    return Sim(graph, trips, profiles, params, **kw)
