"""ctypes wrapper of oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.

Marshals the synth scenario dicts (graph / trips / profiles / params) into the
oracle's own C structs (oracle.h).  Nothing here computes the model.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
# scripts/oracle_mutations.py points this at a deliberately broken build
_LIB_OVERRIDE = os.environ.get("ORACLE_LIB_OVERRIDE")


def lib_path():
    return _LIB


def build(force=False):
    """Compile the oracle (plain g++, fp64, no FMA contraction)."""
    if not force and os.path.exists(_LIB) and \
            os.path.getmtime(_LIB) >= max(os.path.getmtime(_SRC),
                                          os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        return _LIB
    cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math",
           "-fPIC", "-shared", "-o", _LIB, _SRC]
    subprocess.check_call(cmd)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        if _LIB_OVERRIDE:
            _lib = C.CDLL(_LIB_OVERRIDE)
        else:
            build()
            _lib = C.CDLL(_LIB)
        _lib.or_create.restype = C.c_void_p
        _lib.or_create.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p, C.c_int32]
        for f in ("or_destroy",):
            getattr(_lib, f).argtypes = [C.c_void_p]
        _lib.or_step.argtypes = [C.c_void_p, C.c_int32]
        _lib.or_read_state.argtypes = [C.c_void_p, C.c_void_p]
        _lib.or_load_state.argtypes = [C.c_void_p, C.c_void_p]
        _lib.or_lane_order.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_read_decisions.argtypes = [C.c_void_p, C.c_void_p]
        _lib.or_read_metrics.argtypes = [C.c_void_p, C.c_void_p]
        _lib.or_lane_stats.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_set_signal_phase.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        _lib.or_set_lane_direction.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        _lib.or_set_signal_policy.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        _lib.or_set_signal_duration.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        _lib.or_set_vehicle_route.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_float]
        _lib.or_set_lane_max_speed.argtypes = [C.c_void_p, C.c_int32, C.c_float]
        _lib.or_set_lane_restriction.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        _lib.or_road_avg_speed.argtypes = [C.c_void_p, C.c_void_p]
        _lib.or_philox4x32_10.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_u53.restype = C.c_double
        _lib.or_u53.argtypes = [C.c_uint64, C.c_int32, C.c_int32]
        _lib.or_idm.restype = C.c_double
        _lib.or_idm.argtypes = [C.c_double] * 2 + [C.c_int32] + [C.c_double] * 7
        _lib.or_p_lc.restype = C.c_double
        _lib.or_p_lc.argtypes = [C.c_double]
    return _lib


P = C.c_void_p


class _Graph(C.Structure):
    _fields_ = [("n_lanes", C.c_int32), ("n_roads", C.c_int32), ("n_junctions", C.c_int32)] + \
        [(n, P) for n in ("lane_length", "lane_max_speed", "lane_road", "lane_junction",
                          "lane_left", "lane_right", "succ_offsets", "succ_lanes",
                          "lane_turn", "lane_kind", "tidal_partner", "lane_dir0",
                          "road_lane_offsets", "road_lanes", "junc_lane_offsets",
                          "junc_lanes", "junc_phase_offsets", "phase_green",
                          "phase_green_steps", "junc_policy", "junc_offset_steps")]


class _Trips(C.Structure):
    _fields_ = [("n_trips", C.c_int32)] + \
        [(n, P) for n in ("depart_step", "on_network_at_t0", "route_offsets", "route_roads",
                          "start_lane", "start_s", "start_v", "end_s", "profile")]


class _Params(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_profiles", C.c_int32), ("profiles", P),
                ("politeness", C.c_float), ("b_hard", C.c_float), ("b_safe", C.c_float),
                ("v_wait", C.c_float), ("queue_zone_m", C.c_float),
                ("yellow_steps", C.c_int32), ("lookahead_lanes", C.c_int32),
                ("store_fp32", C.c_int32), ("reverse_order", C.c_int32),
                ("max_pressure_period", C.c_int32)]


class _State(C.Structure):
    _fields_ = [("t", C.c_int32)] + [(n, P) for n in (
        "status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time", "s", "v",
        "junc_policy", "junc_phase", "junc_elapsed", "junc_yellow_left", "junc_pending",
        "junc_remaining", "lane_dir", "lane_signal")]


class _Dec(C.Structure):
    _fields_ = [(n, P) for n in ("leader_vid", "leader_hops", "phantom", "old_follower_vid",
                                 "side_vid", "lc", "handoffs", "accel", "finished", "inserted")]


class _Metrics(C.Structure):
    _fields_ = [("t", C.c_int32)] + [(n, C.c_int64) for n in (
        "n_pending", "n_driving", "n_finished", "vehicle_steps", "sum_travel_steps",
        "sum_wait_steps_finished", "sum_depart_delay", "n_lane_changes", "n_handoffs",
        "n_inserted", "sum_time_driving")]


_GRAPH_DT = dict(lane_length=np.float32, lane_max_speed=np.float32, lane_road=np.int32,
                 lane_junction=np.int32, lane_left=np.int32, lane_right=np.int32,
                 succ_offsets=np.int32, succ_lanes=np.int32, lane_turn=np.uint8,
                 lane_kind=np.uint8, tidal_partner=np.int32, lane_dir0=np.uint8,
                 road_lane_offsets=np.int32, road_lanes=np.int32,
                 junc_lane_offsets=np.int32, junc_lanes=np.int32,
                 junc_phase_offsets=np.int32, phase_green=np.uint8,
                 phase_green_steps=np.int32, junc_policy=np.uint8,
                 junc_offset_steps=np.int32)
_TRIP_DT = dict(depart_step=np.int32, on_network_at_t0=np.uint8, route_offsets=np.int32,
                route_roads=np.int32, start_lane=np.int32, start_s=np.float32,
                start_v=np.float32, end_s=np.float32, profile=np.uint8)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """One oracle simulation instance (fp64, serial)."""

    def __init__(self, scen, store_fp32=False, reverse_order=False, lookahead=None):
        lib = _load()
        self._keep = []
        g = {k: np.ascontiguousarray(scen.graph[k], dtype=dt) for k, dt in _GRAPH_DT.items()}
        tr = {k: np.ascontiguousarray(scen.trips[k], dtype=dt) for k, dt in _TRIP_DT.items()}
        self._keep += [g, tr]
        self.n_lanes = int(g["lane_length"].shape[0])
        self.n_roads = int(g["road_lane_offsets"].shape[0] - 1)
        self.n_junctions = int(g["junc_lane_offsets"].shape[0] - 1)
        self.n = int(tr["depart_step"].shape[0])
        G = _Graph(self.n_lanes, int(g["road_lane_offsets"].shape[0] - 1), self.n_junctions,
                   *[_ptr(g[n]) for n, _ in _Graph._fields_[3:]])
        T = _Trips(self.n, *[_ptr(tr[n]) for n, _ in _Trips._fields_[1:]])
        prof = np.ascontiguousarray(scen.profiles, dtype=np.float32)
        self._keep.append(prof)
        p = scen.params
        Pm = _Params(p["seed"], prof.shape[0], _ptr(prof), p["politeness"], p["b_hard"],
                     p["b_safe"], p["v_wait"], p["queue_zone_m"], p["yellow_steps"],
                     p["lookahead_lanes"] if lookahead is None else lookahead,
                     int(store_fp32), int(reverse_order), int(p.get("max_pressure_period", 30)))
        err = C.create_string_buffer(512)
        self.h = lib.or_create(C.byref(G), C.byref(T), C.byref(Pm), err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        self.lib = lib

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.or_destroy(self.h)
            self.h = None

    def step(self, n=1):
        self.lib.or_step(self.h, n)

    def _state_buffers(self):
        n, nj, nl = self.n, self.n_junctions, self.n_lanes
        return dict(status=np.zeros(n, np.uint8), lane=np.zeros(n, np.int32),
                    cursor=np.zeros(n, np.int32), wait_steps=np.zeros(n, np.int32),
                    insert_time=np.zeros(n, np.int32), arrive_time=np.zeros(n, np.int32),
                    s=np.zeros(n, np.float64), v=np.zeros(n, np.float64),
                    junc_policy=np.zeros(nj, np.uint8), junc_phase=np.zeros(nj, np.int32),
                    junc_elapsed=np.zeros(nj, np.int32), junc_yellow_left=np.zeros(nj, np.int32),
                    junc_pending=np.zeros(nj, np.int32), junc_remaining=np.zeros(nj, np.int32),
                    lane_dir=np.zeros(nl, np.uint8),
                    lane_signal=np.zeros(nl, np.uint8))

    def read_state(self):
        b = self._state_buffers()
        st = _State(0, *[_ptr(b[n]) for n, _ in _State._fields_[1:]])
        self.lib.or_read_state(self.h, C.byref(st))
        b["t"] = st.t
        return b

    def load_state(self, state):
        b = self._state_buffers()
        for k in b:
            if k == "junc_remaining" and k not in state:
                b[k][:] = -1                                   # no set_tl_duration timer
                continue
            b[k][:] = np.asarray(state[k]).astype(b[k].dtype)
        st = _State(int(state["t"]), *[_ptr(b[n]) for n, _ in _State._fields_[1:]])
        self.lib.or_load_state(self.h, C.byref(st))

    def lane_order(self):
        off = np.zeros(self.n_lanes + 1, np.int32)
        vids = np.zeros(max(self.n, 1), np.int32)
        self.lib.or_lane_order(self.h, _ptr(off), _ptr(vids))
        return off, vids[:off[-1]]

    def decisions(self):
        n = self.n
        b = dict(leader_vid=np.full(n, -1, np.int32), leader_hops=np.full(n, -1, np.int8),
                 phantom=np.zeros(n, np.int8), old_follower_vid=np.full(n, -1, np.int32),
                 side_vid=np.full(4 * n, -1, np.int32), lc=np.zeros(n, np.int8),
                 handoffs=np.zeros(n, np.int8), accel=np.zeros(n, np.float64),
                 finished=np.zeros(n, np.int8), inserted=np.zeros(n, np.int8))
        d = _Dec(*[_ptr(b[nm]) for nm, _ in _Dec._fields_])
        self.lib.or_read_decisions(self.h, C.byref(d))
        b["side_vid"] = b["side_vid"].reshape(n, 4)
        return b

    def metrics(self):
        m = _Metrics()
        self.lib.or_read_metrics(self.h, C.byref(m))
        out = {n: getattr(m, n) for n, _ in _Metrics._fields_}
        out["att_finished"] = out["sum_travel_steps"] / out["n_finished"] if out["n_finished"] else 0.0
        # ATT over all vehicles ("the average time taken by all vehicles"; ledger L27):
        # finished trips' travel times and the time so far of the trips in progress
        n_all = out["n_finished"] + out["n_driving"]
        out["att_all"] = (out["sum_travel_steps"] + out["sum_time_driving"]) / n_all if n_all else 0.0
        return out

    def lane_stats(self):
        c = np.zeros(self.n_lanes, np.int32)
        w = np.zeros(self.n_lanes, np.int32)
        self.lib.or_lane_stats(self.h, _ptr(c), _ptr(w))
        return c, w

    def set_signal_phase(self, j, p):
        return self.lib.or_set_signal_phase(self.h, int(j), int(p))

    def set_lane_direction(self, lane, d):
        return self.lib.or_set_lane_direction(self.h, int(lane), int(d))

    def set_signal_policy(self, j, policy):
        return self.lib.or_set_signal_policy(self.h, int(j), int(policy))

    def set_signal_duration(self, j, steps):
        return self.lib.or_set_signal_duration(self.h, int(j), int(steps))

    def set_vehicle_route(self, vid, roads, end_s):
        r = np.ascontiguousarray(roads, np.int32)
        return self.lib.or_set_vehicle_route(self.h, int(vid), len(r), _ptr(r), float(end_s))

    def set_lane_max_speed(self, lane, v):
        return self.lib.or_set_lane_max_speed(self.h, int(lane), float(v))

    def set_lane_restriction(self, lane, flag):
        return self.lib.or_set_lane_restriction(self.h, int(lane), int(flag))

    def road_avg_speed(self):
        out = np.zeros(self.n_roads, np.float64)
        self.lib.or_road_avg_speed(self.h, _ptr(out))
        return out


def philox4x32_10(ctr, key):
    lib = _load()
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib.or_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o


def u53(seed, vid, t):
    return _load().or_u53(seed, vid, t)


def idm(v, v0, has_leader, gap, dv, a_max=2.0, a_comf=3.0, T=1.5, s0=2.0, b_hard=8.0):
    return _load().or_idm(v, v0, int(has_leader), gap, dv, a_max, a_comf, T, s0, b_hard)


def p_lc(u):
    return _load().or_p_lc(u)
