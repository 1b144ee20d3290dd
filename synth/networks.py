"""Seeded synthetic lane graphs + trips shaped like the paper's workloads.

Config recipes follow SURVEY §8(d) (C1 ring, C2 4x4 signalised grid, C3 20x20
grid with dynamic + tidal lanes, C4 city-like perturbed grid, C5 tiles).  The
paper's own performance workloads (Roadnet-S/M/L) are CBLab
datasets that are not available; these generators reproduce their shape
(grid-like city graphs, ~3.5 roads per junction, signalised 4-approach
junctions, shortest-time routes) with seeded synthetic data.

Nothing here implements the model (no car following, lane changing, signals
or ordering): only graph construction, routing for demand generation (which
is an input to the method) and placement.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np

TURN_STRAIGHT, TURN_LEFT, TURN_RIGHT = 0, 1, 2
KIND_NORMAL, KIND_DYNAMIC, KIND_TIDAL = 0, 1, 2
POLICY_NONE, POLICY_FIXED, POLICY_MANUAL, POLICY_MAXP = 0, 1, 2, 3

# heading index: 0 = +x (E), 1 = +y (N), 2 = -x (W), 3 = -y (S)
_DXY = [(1, 0), (0, 1), (-1, 0), (0, -1)]


def default_profiles():
    """Profile table rows (a_max, a_comf, T, s0, v_max, length) — ledger L4."""
    return np.array([[2.0, 3.0, 1.5, 2.0, 16.667, 5.0]], dtype=np.float32)


def city_profiles():
    """car / van / bus."""
    return np.array([[2.0, 3.0, 1.5, 2.0, 33.3, 5.0],
                     [1.5, 3.0, 1.5, 2.0, 27.8, 7.0],
                     [1.0, 3.0, 1.5, 2.0, 22.2, 12.0]], dtype=np.float32)


def default_params(seed=1):
    return dict(seed=int(seed), dt=1.0, politeness=0.1, b_hard=8.0, b_safe=4.0,
                v_wait=0.1, queue_zone_m=100.0, yellow_steps=3,
                lookahead_lanes=2, max_pressure_period=30)


@dataclass
class Scenario:
    name: str
    graph: dict
    trips: dict
    profiles: np.ndarray
    params: dict
    meta: dict = field(default_factory=dict)

    @property
    def n_lanes(self):
        return int(self.graph["lane_length"].shape[0])

    @property
    def n_trips(self):
        return int(self.trips["depart_step"].shape[0])


def save_scenario(scen, path):
    """Cache a scenario as .npz (graph / trips / profiles / params)."""
    d = {f"g_{k}": v for k, v in scen.graph.items()}
    d.update({f"t_{k}": v for k, v in scen.trips.items()})
    d["profiles"] = scen.profiles
    d["params_json"] = np.frombuffer(__import__("json").dumps(scen.params).encode(), np.uint8)
    d["name"] = np.frombuffer(scen.name.encode(), np.uint8)
    np.savez(path, **d)


def load_scenario(path):
    import json
    z = np.load(path)
    g = {k[2:]: z[k] for k in z.files if k.startswith("g_")}
    t = {k[2:]: z[k] for k in z.files if k.startswith("t_")}
    return Scenario(bytes(z["name"]).decode(), g, t, z["profiles"],
                    json.loads(bytes(z["params_json"]).decode()))


class NetBuilder:
    """Incremental lane-graph builder producing the sim_graph CSR arrays."""

    def __init__(self):
        self.lane_length, self.lane_vmax = [], []
        self.lane_road, self.lane_junc = [], []
        self.lane_left, self.lane_right = [], []
        self.lane_turn, self.lane_kind, self.lane_dir0 = [], [], []
        self.tidal_partner = []
        self.succ = []
        self.road_lanes = []          # list of lists, leftmost first
        self.road_meta = []           # (from_junction, to_junction, heading)
        self.junc_lanes = []          # list of lists
        self.junc_xy = []
        self.junc_phases = []         # list of (list of green sets, durations)
        self.junc_policy = []
        self.junc_offset = []
        self.jl_src = {}              # junction lane -> (in road, movement)

    # -- entities ---------------------------------------------------------
    def add_junction(self, x=0.0, y=0.0, policy=POLICY_FIXED, offset=0):
        self.junc_lanes.append([])
        self.junc_xy.append((x, y))
        self.junc_phases.append(([], []))
        self.junc_policy.append(policy)
        self.junc_offset.append(int(offset))
        return len(self.junc_lanes) - 1

    def _new_lane(self, length, vmax, road=-1, junc=-1, turn=0, kind=0, dir0=0):
        self.lane_length.append(float(length))
        self.lane_vmax.append(float(vmax))
        self.lane_road.append(road)
        self.lane_junc.append(junc)
        self.lane_left.append(-1)
        self.lane_right.append(-1)
        self.lane_turn.append(turn)
        self.lane_kind.append(kind)
        self.lane_dir0.append(dir0)
        self.tidal_partner.append(-1)
        self.succ.append([])
        return len(self.lane_length) - 1

    def add_road(self, n_lanes, length, vmax, kinds=None, src=-1, dst=-1,
                 heading=-1):
        rid = len(self.road_lanes)
        kinds = kinds or [KIND_NORMAL] * n_lanes
        ids = [self._new_lane(length, vmax, road=rid, kind=kinds[i])
               for i in range(n_lanes)]
        for i in range(n_lanes - 1):
            self.lane_right[ids[i]] = ids[i + 1]
            self.lane_left[ids[i + 1]] = ids[i]
        self.road_lanes.append(ids)
        self.road_meta.append((src, dst, heading))
        return rid

    def connect_direct(self, lane_from, lane_to):
        """Road lane -> road lane without a junction (ledger L33)."""
        self.succ[lane_from].append(lane_to)

    def connect(self, junc, lane_from, lane_to, turn, length, vmax):
        jl = self._new_lane(length, vmax, junc=junc, turn=turn)
        self.succ[lane_from].append(jl)
        self.succ[jl].append(lane_to)
        self.junc_lanes[junc].append(jl)
        self.jl_src[jl] = (self.lane_road[lane_from], turn)
        return jl

    def set_phases(self, junc, green_sets, durations):
        self.junc_phases[junc] = (list(green_sets), list(durations))

    # -- output -----------------------------------------------------------
    def graph(self):
        nl = len(self.lane_length)
        succ_off = np.zeros(nl + 1, np.int32)
        succ_off[1:] = np.cumsum([len(s) for s in self.succ])
        succ = np.array([x for s in self.succ for x in s], np.int32)
        road_off = np.zeros(len(self.road_lanes) + 1, np.int32)
        road_off[1:] = np.cumsum([len(r) for r in self.road_lanes])
        road_lanes = np.array([x for r in self.road_lanes for x in r], np.int32)
        jl_off = np.zeros(len(self.junc_lanes) + 1, np.int32)
        jl_off[1:] = np.cumsum([len(j) for j in self.junc_lanes])
        junc_lanes = np.array([x for j in self.junc_lanes for x in j], np.int32)
        ph_off = np.zeros(len(self.junc_lanes) + 1, np.int32)
        ph_off[1:] = np.cumsum([len(p[0]) for p in self.junc_phases])
        green, steps = [], []
        for j, (sets, durs) in enumerate(self.junc_phases):
            lanes = self.junc_lanes[j]
            for gs, d in zip(sets, durs):
                green.extend(1 if l in gs else 0 for l in lanes)
                steps.append(int(d))
        return dict(
            lane_length=np.array(self.lane_length, np.float32),
            lane_max_speed=np.array(self.lane_vmax, np.float32),
            lane_road=np.array(self.lane_road, np.int32),
            lane_junction=np.array(self.lane_junc, np.int32),
            lane_left=np.array(self.lane_left, np.int32),
            lane_right=np.array(self.lane_right, np.int32),
            succ_offsets=succ_off, succ_lanes=succ,
            lane_turn=np.array(self.lane_turn, np.uint8),
            lane_kind=np.array(self.lane_kind, np.uint8),
            tidal_partner=np.array(self.tidal_partner, np.int32),
            lane_dir0=np.array(self.lane_dir0, np.uint8),
            road_lane_offsets=road_off, road_lanes=road_lanes,
            junc_lane_offsets=jl_off, junc_lanes=junc_lanes,
            junc_phase_offsets=ph_off,
            phase_green=np.array(green, np.uint8),
            phase_green_steps=np.array(steps, np.int32),
            junc_policy=np.array(self.junc_policy, np.uint8),
            junc_offset_steps=np.array(self.junc_offset, np.int32),
        )

    # -- road-level connectivity (for demand generation only) -------------
    def road_successors(self):
        """road -> sorted list of roads reachable through one lane connection."""
        out = [set() for _ in self.road_lanes]
        for r, lanes in enumerate(self.road_lanes):
            for l in lanes:
                for j in self.succ[l]:
                    tr = self.lane_road[j] if self.lane_road[j] >= 0 \
                        else self.lane_road[self.succ[j][0]]
                    out[r].add(tr)
        return [sorted(s) for s in out]

    def lanes_toward(self, road, next_road, static_only=True):
        """Lanes of `road` with a successor toward `next_road` (NORMAL lanes
        preferred; used to pick trip start lanes consistent with the first turn)."""
        res = []
        for l in self.road_lanes[road]:
            if static_only and self.lane_kind[l] != KIND_NORMAL:
                continue
            for j in self.succ[l]:
                tr = self.lane_road[j] if self.lane_road[j] >= 0 \
                    else self.lane_road[self.succ[j][0]]
                if tr == next_road:
                    res.append(l)
                    break
        return res


# ---------------------------------------------------------------------------
# C1 ring
# ---------------------------------------------------------------------------
def ring(n_vehicles=20, length=1000.0, laps=40, vmax=16.667, seed=1,
         spacing=None, n_lanes=1, profiles=None, speeds=None):
    """C1: one road whose lane(s) succeed themselves (ledger L33).

    Vehicles start at rest, evenly spaced (s = spacing*k), on_network_at_t0.
    """
    b = NetBuilder()
    r = b.add_road(n_lanes, length, vmax)
    for l in b.road_lanes[r]:
        b.connect_direct(l, l)
    spacing = length * n_lanes / n_vehicles if spacing is None else spacing
    n = n_vehicles
    lanes = np.array([b.road_lanes[r][k % n_lanes] for k in range(n)], np.int32)
    s = np.array([(spacing * (k // n_lanes)) % length for k in range(n)],
                 np.float32)
    # keep s in (0, L]: a front bumper at 0 would put the rear behind the lane
    s = np.where(s <= 0, np.float32(length), s).astype(np.float32)
    v = np.zeros(n, np.float32) if speeds is None else \
        np.asarray(speeds, np.float32)
    trips = dict(
        depart_step=np.zeros(n, np.int32),
        on_network_at_t0=np.ones(n, np.uint8),
        route_offsets=(np.arange(n + 1) * laps).astype(np.int32),
        route_roads=np.full(n * laps, r, np.int32),
        start_lane=lanes, start_s=s, start_v=v,
        end_s=np.full(n, length, np.float32),
        profile=np.zeros(n, np.uint8))
    prof = default_profiles() if profiles is None else profiles
    return Scenario("ring", b.graph(), trips, prof, default_params(seed),
                    meta=dict(builder=b))


# ---------------------------------------------------------------------------
# grids (C2, C3) and the city (C4)
# ---------------------------------------------------------------------------
def _movement_targets(n_in, tidal_in, dyn_in, n_out, tidal_out, turn):
    """(in lane index, out lane index) pairs for one movement.

    Junction lanes fan out to the exit lane of the same index and its
    neighbours (a vehicle picks its exit lane inside the junction, ledger L24);
    LEFT leaves from the leftmost regular lane (and the tidal / dynamic lanes),
    RIGHT from the rightmost lane.
    """
    off_in, off_out = int(tidal_in), int(tidal_out)
    lo, hi = off_out, n_out - 1            # regular exit lanes

    def fan(j):
        return [x for x in (j - 1, j, j + 1) if lo <= x <= hi]
    pairs = []
    if turn == TURN_STRAIGHT:
        for i in range(n_in):
            if i < off_in:                  # tidal lane -> tidal exit (+ leftmost regular)
                outs = ([0] if tidal_out else []) + [lo]
            else:
                outs = fan(min(max(i - off_in + off_out, lo), hi))
            pairs += [(i, o) for o in outs]
    elif turn == TURN_LEFT:
        srcs = sorted({0, off_in} | ({dyn_in} if dyn_in >= 0 else set()))
        for i in srcs:
            if i >= n_in:
                continue
            outs = ([0] if (i < off_in and tidal_out) else []) + \
                [x for x in (lo, lo + 1) if x <= hi]
            pairs += [(i, o) for o in outs]
    else:
        pairs += [(n_in - 1, o) for o in (hi, hi - 1) if o >= lo]
    return pairs


_JL_LEN = {TURN_STRAIGHT: 20.0, TURN_LEFT: 25.0, TURN_RIGHT: 10.0}


def _build_junction_lanes(b, junc, in_roads, out_roads, road_info):
    """in_roads/out_roads: heading -> road id (heading of travel)."""
    green = [set(), set(), set(), set()]   # NS S+R, NS L, EW S+R, EW L
    for h, rin in sorted(in_roads.items()):
        n_in, tid_in, dyn_in, vin = road_info[rin]
        for turn, hout in ((TURN_LEFT, (h + 1) % 4), (TURN_STRAIGHT, h),
                           (TURN_RIGHT, (h + 3) % 4)):
            rout = out_roads.get(hout)
            if rout is None:
                continue
            n_out, tid_out, _, vout = road_info[rout]
            pairs = _movement_targets(n_in, tid_in, dyn_in, n_out, tid_out,
                                      turn)
            for i, o in pairs:
                jl = b.connect(junc, b.road_lanes[rin][i], b.road_lanes[rout][o],
                               turn, _JL_LEN[turn], min(vin, vout))
                ns = h in (1, 3)
                phase = (0 if ns else 2) + (1 if turn == TURN_LEFT else 0)
                green[phase].add(jl)
    return green


def _grid_core(rows, cols, spacing, lane_fn, vmax_fn, rng, jitter=0.0,
               stubs=True, stub_len=300.0, tidal=False, dynamic=False,
               remove_frac=0.0, policy=POLICY_FIXED, phase_steps=(30, 15, 30, 15),
               offsets=None):
    b = NetBuilder()
    pos = {}
    jid = {}
    for i in range(rows):
        for j in range(cols):
            x = j * spacing + (rng.uniform(-jitter, jitter) * spacing if jitter else 0.0)
            y = i * spacing + (rng.uniform(-jitter, jitter) * spacing if jitter else 0.0)
            pos[(i, j)] = (x, y)
            off = 0 if offsets is None else int(offsets(rng))
            jid[(i, j)] = b.add_junction(x, y, policy, off)
    # undirected junction pairs
    pairs = []
    for i in range(rows):
        for j in range(cols):
            if j + 1 < cols:
                pairs.append(((i, j), (i, j + 1)))
            if i + 1 < rows:
                pairs.append(((i, j), (i + 1, j)))
    keep = set(pairs)
    if remove_frac > 0:
        deg = {k: 0 for k in pos}
        for a, c in pairs:
            deg[a] += 1
            deg[c] += 1
        order = rng.permutation(len(pairs))
        target = int(remove_frac * len(pairs))
        removed = 0
        for idx in order:
            if removed >= target:
                break
            a, c = pairs[idx]
            if deg[a] <= 2 or deg[c] <= 2:
                continue
            keep.discard((a, c))
            deg[a] -= 1
            deg[c] -= 1
            removed += 1
        if not _connected(pos.keys(), keep):
            raise RuntimeError("removal disconnected the grid; use another seed")
    road_info = {}
    in_roads = {k: {} for k in pos}
    out_roads = {k: {} for k in pos}

    def heading(a, c):
        di, dj = c[0] - a[0], c[1] - a[1]
        return {(0, 1): 0, (1, 0): 1, (0, -1): 2, (-1, 0): 3}[(di, dj)]

    def make_road(a, c, h, length, n_reg, vmax, has_tidal):
        kinds = []
        if has_tidal:
            kinds.append(KIND_TIDAL)
        dyn_idx = -1
        for k in range(n_reg):
            if dynamic and n_reg >= 3 and k == n_reg // 2:
                dyn_idx = len(kinds)
                kinds.append(KIND_DYNAMIC)
            else:
                kinds.append(KIND_NORMAL)
        src = jid[a] if a is not None else -1
        dst = jid[c] if c is not None else -1
        r = b.add_road(len(kinds), length, vmax, kinds, src, dst, h)
        road_info[r] = (len(kinds), has_tidal, dyn_idx, vmax)
        return r

    tidal_pairs = []
    for (a, c) in sorted(keep):
        ln = float(np.hypot(pos[a][0] - pos[c][0], pos[a][1] - pos[c][1]))
        n_reg = lane_fn(a, c)
        vm = vmax_fn(a, c)
        r1 = make_road(a, c, heading(a, c), ln, n_reg, vm, tidal)
        r2 = make_road(c, a, heading(c, a), ln, n_reg, vm, tidal)
        out_roads[a][heading(a, c)] = r1
        in_roads[c][heading(a, c)] = r1
        out_roads[c][heading(c, a)] = r2
        in_roads[a][heading(c, a)] = r2
        if tidal:
            tidal_pairs.append((r1, r2))
    sources, sinks = [], []
    if stubs:
        for (i, j) in sorted(pos):
            for h, (dx, dy) in enumerate(_DXY):
                ni, nj = i + dy, j + dx
                if 0 <= ni < rows and 0 <= nj < cols:
                    continue
                n_reg = lane_fn((i, j), None)
                vm = vmax_fn((i, j), None)
                r_out = make_road((i, j), None, h, stub_len, n_reg, vm, False)
                r_in = make_road(None, (i, j), (h + 2) % 4, stub_len, n_reg, vm,
                                 False)
                out_roads[(i, j)][h] = r_out
                in_roads[(i, j)][(h + 2) % 4] = r_in
                sources.append((r_in, h))
                sinks.append((r_out, h))
    for k in sorted(pos):
        green = _build_junction_lanes(b, jid[k], in_roads[k], out_roads[k],
                                      road_info)
        b.set_phases(jid[k], green, phase_steps)
    for r1, r2 in tidal_pairs:
        l1, l2 = b.road_lanes[r1][0], b.road_lanes[r2][0]
        b.tidal_partner[l1], b.tidal_partner[l2] = l2, l1
        b.lane_dir0[l1], b.lane_dir0[l2] = 0, 1     # r1's lane open (FORWARD)
    return b, sources, sinks


def _connected(nodes, edges):
    nodes = list(nodes)
    adj = {n: [] for n in nodes}
    for a, c in edges:
        adj[a].append(c)
        adj[c].append(a)
    seen = {nodes[0]}
    st = [nodes[0]]
    while st:
        n = st.pop()
        for m in adj[n]:
            if m not in seen:
                seen.add(m)
                st.append(m)
    return len(seen) == len(nodes)


def _road_costs(b):
    g = b.graph()
    L = g["lane_length"]
    V = g["lane_max_speed"]
    return np.array([float(L[ls[0]]) / float(V[ls[0]]) for ls in b.road_lanes])


def _dijkstra_tree(succ, cost, src):
    n = len(succ)
    dist = np.full(n, np.inf)
    prev = np.full(n, -1, np.int64)
    dist[src] = 0.0
    pq = [(0.0, src)]
    while pq:
        d, u = heapq.heappop(pq)
        if d > dist[u]:
            continue
        for w in succ[u]:
            nd = d + cost[w]
            if nd < dist[w] - 1e-9:
                dist[w] = nd
                prev[w] = u
                heapq.heappush(pq, (nd, w))
    return prev


def _path(prev, src, dst):
    p = [dst]
    while p[-1] != src:
        q = prev[p[-1]]
        if q < 0:
            return None
        p.append(int(q))
    return p[::-1]


def _trip_arrays(routes, start_lane, start_s, start_v, end_s, depart, on_net,
                 profile):
    n = len(routes)
    off = np.zeros(n + 1, np.int32)
    off[1:] = np.cumsum([len(r) for r in routes])
    return dict(
        depart_step=np.asarray(depart, np.int32),
        on_network_at_t0=np.asarray(on_net, np.uint8),
        route_offsets=off,
        route_roads=np.array([x for r in routes for x in r], np.int32),
        start_lane=np.asarray(start_lane, np.int32),
        start_s=np.asarray(start_s, np.float32),
        start_v=np.asarray(start_v, np.float32),
        end_s=np.asarray(end_s, np.float32),
        profile=np.asarray(profile, np.uint8))


def grid(rows=4, cols=4, road_len=300.0, lanes=2, n_trips=5000,
         depart_window=1800, seed=2, vmax=16.667, tidal=False, dynamic=False,
         policy=POLICY_FIXED, start_s=30.0, min_hops=0, phase_steps=(30, 15, 30, 15)):
    """C2 (defaults) / C3 (rows=cols=20, road_len=500, lanes=3, tidal, dynamic).

    Trips: source stub -> sink stub on a different side, shortest free-flow
    time route, start lane consistent with the first turn, departures uniform
    in [0, depart_window) (P:300-307 shape).
    """
    rng = np.random.default_rng(seed)
    b, sources, sinks = _grid_core(rows, cols, road_len, lambda a, c: lanes,
                                   lambda a, c: vmax, rng, stubs=True,
                                   stub_len=road_len, tidal=tidal,
                                   dynamic=dynamic, policy=policy,
                                   phase_steps=phase_steps)
    succ = b.road_successors()
    cost = _road_costs(b)
    trees = {}
    routes, sl, ss, es, dep = [], [], [], [], []
    lane_len = b.graph()["lane_length"]
    while len(routes) < n_trips:
        si = int(rng.integers(len(sources)))
        src, sh = sources[si]
        cands = [k for k, (r, h) in enumerate(sinks) if h != sh]
        dst, _ = sinks[cands[int(rng.integers(len(cands)))]]
        if src not in trees:
            trees[src] = _dijkstra_tree(succ, cost, src)
        p = _path(trees[src], src, dst)
        if p is None or len(p) < 2 or len(p) - 2 < min_hops:
            continue
        ok = b.lanes_toward(p[0], p[1])
        if not ok:
            continue
        routes.append(p)
        sl.append(ok[int(rng.integers(len(ok)))])
        ss.append(start_s)
        es.append(float(lane_len[b.road_lanes[p[-1]][0]]))
        dep.append(int(rng.integers(depart_window)))
    n = len(routes)
    trips = _trip_arrays(routes, sl, ss, np.zeros(n), es, dep, np.zeros(n),
                         np.zeros(n))
    return Scenario(f"grid{rows}x{cols}", b.graph(), trips, default_profiles(),
                    default_params(seed),
                    meta=dict(builder=b, sources=sources, sinks=sinks))


def _random_walks(b, succ_roads, start_roads, n_roads, rng):
    """Vectorised biased random walks (straight 0.6, left 0.2, right 0.2, no
    U-turn) of n_roads roads from each start road; a walk stops at a dead end."""
    meta = b.road_meta
    nr = len(meta)
    cand = np.full((nr, 3), -1, np.int64)
    w = np.zeros((nr, 3))
    for r in range(nr):
        h = meta[r][2]
        k = 0
        for r2 in succ_roads[r]:
            h2 = meta[r2][2]
            if h2 == (h + 2) % 4 or k >= 3:
                continue
            cand[r, k] = r2
            w[r, k] = 0.6 if h2 == h else 0.2
            k += 1
    tot = w.sum(1, keepdims=True)
    cw = np.cumsum(np.where(tot > 0, w / np.where(tot > 0, tot, 1), 0), axis=1)
    n = len(start_roads)
    routes = np.full((n, n_roads), -1, np.int64)
    routes[:, 0] = start_roads
    alive = np.ones(n, bool)
    for s in range(1, n_roads):
        cur = routes[:, s - 1]
        u = rng.random(n)
        pick = (u[:, None] >= cw[np.maximum(cur, 0)]).sum(1)
        pick = np.minimum(pick, 2)
        nxt = cand[np.maximum(cur, 0), pick]
        alive &= (cur >= 0) & (tot[np.maximum(cur, 0), 0] > 0) & (nxt >= 0)
        routes[:, s] = np.where(alive, nxt, -1)
    lens = (routes >= 0).sum(1)
    return routes, lens


def _place_on_lanes(lane_ids, lane_len, n_vehicles, prof_len, profile_of, rng,
                    s0=2.0):
    """Uniform placement over road lanes, non-overlapping with gap >= s0."""
    cap = lane_len[lane_ids]
    p = cap / cap.sum()
    counts = rng.multinomial(n_vehicles, p)
    order = rng.permutation(n_vehicles)
    lanes_out = np.empty(n_vehicles, np.int32)
    s_out = np.empty(n_vehicles, np.float32)
    k = 0
    spill = 0
    plan = []
    for li, lane in enumerate(lane_ids):
        c = int(counts[li])
        if c == 0:
            continue
        L = float(lane_len[lane])
        vids = order[k:k + c]
        k += c
        lens = prof_len[profile_of[vids]]
        need = float(lens.sum()) + s0 * (c - 1)
        while need > L - 1.0 and c > 0:
            spill += 1
            c -= 1
            lens = lens[:c]
            need = float(lens.sum()) + s0 * max(c - 1, 0)
        plan.append((lane, vids[:c], lens, L - need - 1.0))
        if len(vids) > c:
            plan.append((None, vids[c:], None, None))
    pending_spill = []
    for lane, vids, lens, slack in plan:
        if lane is None:
            pending_spill.extend(vids.tolist())
            continue
        c = len(vids)
        cuts = np.sort(rng.uniform(0.0, slack, c)) if slack > 0 else np.zeros(c)
        rear = 0.5
        for idx in range(c):
            extra = cuts[idx] - (cuts[idx - 1] if idx else 0.0)
            rear += extra
            front = rear + float(lens[idx])
            lanes_out[vids[idx]] = lane
            s_out[vids[idx]] = np.float32(front)
            rear = front + s0
    # spill (rare): append at the least occupied lanes' fronts is complex; drop
    keep = np.ones(n_vehicles, bool)
    keep[pending_spill] = False
    return lanes_out, s_out, keep


def city(G=72, spacing=900.0, n_vehicles=2_000_000, seed=4, route_len=40,
         jitter=0.15, remove_frac=0.10, arterial_every=6, arterial_lanes=3):
    """C4: city-like perturbed grid.

    Arterials (every `arterial_every`-th grid line) have `arterial_lanes`
    lanes (3 in C4) at 22.2 m/s,
    other roads 1 or 2 lanes (p = 0.5) at 13.9 m/s.  All vehicles are on the
    network at t = 0, at rest, uniformly over road lanes, with biased random
    walk routes of `route_len` roads (straight 0.6, left 0.2, right 0.2).
    """
    rng = np.random.default_rng(seed)
    pair_lanes = {}

    def is_art(a, c):
        return (a[0] == c[0] and a[0] % arterial_every == 0) or \
               (a[1] == c[1] and a[1] % arterial_every == 0)

    def lane_fn(a, c):
        key = (a, c) if a < c else (c, a)
        if key not in pair_lanes:
            pair_lanes[key] = arterial_lanes if is_art(a, c) else int(rng.integers(1, 3))
        return pair_lanes[key]

    def vmax_fn(a, c):
        return 22.2 if is_art(a, c) else 13.9
    C = 102
    b, _, _ = _grid_core(G, G, spacing, lane_fn, vmax_fn, rng, jitter=jitter,
                         stubs=False, remove_frac=remove_frac,
                         offsets=lambda r: r.integers(C))
    g = b.graph()
    profiles = city_profiles()
    mix = np.array([0.80, 0.15, 0.05])
    profile_of = rng.choice(3, size=n_vehicles, p=mix).astype(np.uint8)
    road_lane_ids = np.where(g["lane_road"] >= 0)[0]
    lanes, s, keep = _place_on_lanes(road_lane_ids, g["lane_length"], n_vehicles,
                                     profiles[:, 5], profile_of, rng)
    succ_roads = b.road_successors()
    idx = np.where(keep)[0]
    r0 = g["lane_road"][lanes[idx]]
    rt, lens = _random_walks(b, succ_roads, r0, route_len, rng)
    n = len(idx)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    flat = rt[rt >= 0]
    last = rt[np.arange(n), lens - 1]
    first_lane_of_road = g["road_lanes"][g["road_lane_offsets"][:-1]]
    end_s = g["lane_length"][first_lane_of_road[last]]
    trips = dict(depart_step=np.zeros(n, np.int32), on_network_at_t0=np.ones(n, np.uint8),
                 route_offsets=off.astype(np.int32), route_roads=flat.astype(np.int32),
                 start_lane=lanes[idx].astype(np.int32), start_s=s[idx].astype(np.float32),
                 start_v=np.zeros(n, np.float32), end_s=end_s.astype(np.float32),
                 profile=profile_of[idx].astype(np.uint8))
    road_dst = np.array([m[1] for m in b.road_meta], np.int64)
    return Scenario(f"city{G}", g, trips, profiles, default_params(seed),
                    meta=dict(builder=b, junc_xy=np.array(b.junc_xy), road_dst=road_dst))


def rcb_partition(scen, world):
    """Recursive coordinate bisection of the roads into `world` parts by the
    coordinates of their downstream junctions, weighted by lane-metres (a road
    travels with its outgoing junction lanes: DESIGN §6).  Input preparation
    for partitioned runs; the library has its own coordinate-free default."""
    g = scen.graph
    xy = np.asarray(scen.meta["junc_xy"], np.float64)[scen.meta["road_dst"]]
    nl = np.diff(g["road_lane_offsets"])
    L = g["lane_length"][g["road_lanes"][g["road_lane_offsets"][:-1]]]
    w = nl * L
    owner = np.zeros(len(nl), np.int32)

    def split(idx, parts, base, depth):
        if parts == 1:
            owner[idx] = base
            return
        ext = xy[idx].max(0) - xy[idx].min(0)
        ax = int(np.argmax(ext))
        order = idx[np.lexsort((idx, xy[idx, ax]))]
        left = parts // 2
        cw = np.cumsum(w[order])
        cut = int(np.searchsorted(cw, cw[-1] * left / parts))
        split(order[:cut], left, base, depth + 1)
        split(order[cut:], parts - left, base + left, depth + 1)

    split(np.arange(len(nl)), world, 0, 0)
    return owner


def tiled_city(tiles_x=1, tiles_y=1, G=50, n_per_tile=1_000_000, seed=5, **kw):
    """C5: a (tiles_x*G) x (tiles_y*G) city with n_per_tile vehicles per G x G
    tile (weak-scaling instance; tiles are the natural GPU partition)."""
    s = city(G=G * max(tiles_x, tiles_y), n_vehicles=n_per_tile * tiles_x * tiles_y,
             seed=seed, **kw) if tiles_x == tiles_y else None
    if s is None:
        raise NotImplementedError("non-square tilings: use city(G=...)")
    s.name = f"tiled{tiles_x}x{tiles_y}_G{G}"
    return s


def pressure_junction(counts, road_len=200.0, vmax=13.9, period=30, spacing=10.0):
    """One MAX_PRESSURE junction with three single-lane approaches A, B, C and
    exits D, E, F; movements A->D and B->E form phase 0, C->F phase 1 (the
    two-phase example of S:336).  `counts` = vehicles initially on
    (A, B, C, D, E, F), at rest, spaced `spacing` m from the far end; each
    vehicle's route ends on its movement's exit road (or on its own exit road).
    Returns (scenario, junction lanes (A->D, B->E, C->F))."""
    b = NetBuilder()
    j = b.add_junction(policy=POLICY_MAXP)
    rid = [b.add_road(1, road_len, vmax, dst=j) for _ in range(3)] + \
          [b.add_road(1, road_len, vmax, src=j) for _ in range(3)]
    lane = [b.road_lanes[r][0] for r in rid]
    jls = [b.connect(j, lane[i], lane[i + 3], TURN_STRAIGHT, 20.0, vmax) for i in range(3)]
    b.set_phases(j, [{jls[0], jls[1]}, {jls[2]}], [period, period])
    routes, sl, ss = [], [], []
    for i, c in enumerate(counts):
        for k in range(int(c)):
            routes.append([rid[i], rid[i + 3]] if i < 3 else [rid[i]])
            sl.append(lane[i])
            ss.append(road_len - 1.0 - spacing * k)
    n = len(routes)
    trips = _trip_arrays(routes, sl, ss, np.zeros(n), [road_len] * n, np.zeros(n),
                         np.ones(n), np.zeros(n))
    params = default_params(1)
    params["max_pressure_period"] = int(period)
    return Scenario("pressure_junction", b.graph(), trips, default_profiles(), params), jls


def batch(scens):
    """NEXT-3 batched environments: the disjoint union of independent
    scenarios as one input (ids offset per environment), plus the per-vehicle
    Philox seed / counter id and per-road group that make each environment
    behave exactly like its standalone run (sim_params.vehicle_seed,
    vehicle_rng_id, road_group).  Input construction only (no model logic).
    The profile table and model parameters of scens[0] apply to all."""
    g0 = scens[0].graph
    out_g = {k: [] for k in g0}
    trips = {k: [] for k in scens[0].trips}
    lo = ro = jo = po = 0
    vseed, rid, rgroup = [], [], []
    for e, sc in enumerate(scens):
        g, tr = sc.graph, sc.trips
        nl, nr = len(g["lane_length"]), len(g["road_lane_offsets"]) - 1
        nj = len(g["junc_lane_offsets"]) - 1
        sh = lambda a, o: np.where(np.asarray(a) >= 0, np.asarray(a) + o, np.asarray(a))
        for k in ("lane_length", "lane_max_speed", "lane_turn", "lane_kind", "lane_dir0",
                  "phase_green", "phase_green_steps", "junc_policy", "junc_offset_steps"):
            out_g[k].append(np.asarray(g[k]))
        out_g["lane_road"].append(sh(g["lane_road"], ro))
        out_g["lane_junction"].append(sh(g["lane_junction"], jo))
        out_g["lane_left"].append(sh(g["lane_left"], lo))
        out_g["lane_right"].append(sh(g["lane_right"], lo))
        out_g["tidal_partner"].append(sh(g["tidal_partner"], lo))
        out_g["succ_lanes"].append(np.asarray(g["succ_lanes"]) + lo)
        out_g["road_lanes"].append(np.asarray(g["road_lanes"]) + lo)
        out_g["junc_lanes"].append(np.asarray(g["junc_lanes"]) + lo)
        for k, base in (("succ_offsets", sum(len(x) for x in out_g["succ_lanes"][:-1])),
                        ("road_lane_offsets", sum(len(x) for x in out_g["road_lanes"][:-1])),
                        ("junc_lane_offsets", sum(len(x) for x in out_g["junc_lanes"][:-1])),
                        ("junc_phase_offsets", po)):
            a = np.asarray(g[k])
            out_g[k].append((a if e == 0 else a[1:]) + base)
        n = len(tr["depart_step"])
        for k in trips:
            if k != "route_offsets":
                trips[k].append(np.asarray(tr[k]))
        trips["route_roads"][-1] = trips["route_roads"][-1] + ro
        trips["start_lane"][-1] = trips["start_lane"][-1] + lo
        ro_base = sum(len(x) for x in trips["route_roads"][:-1])
        a = np.asarray(tr["route_offsets"])
        trips["route_offsets"].append((a if e == 0 else a[1:]) + ro_base)
        vseed += [int(sc.params["seed"])] * n
        rid += list(range(n))
        rgroup += [e] * nr
        lo += nl; ro += nr; jo += nj; po += int(np.asarray(g["junc_phase_offsets"])[-1])
    G = {k: np.concatenate(v).astype(np.asarray(g0[k]).dtype) for k, v in out_g.items()}
    T = {k: np.concatenate(v).astype(np.asarray(scens[0].trips[k]).dtype) for k, v in trips.items()}
    params = dict(scens[0].params)
    params["vehicle_seed"] = np.asarray(vseed, np.uint64)
    params["vehicle_rng_id"] = np.asarray(rid, np.int32)
    params["road_group"] = np.asarray(rgroup, np.int32)
    params["n_groups"] = len(scens)
    return Scenario(f"batch{len(scens)}", G, T, scens[0].profiles, params,
                    meta=dict(env_lanes=[len(s.graph["lane_length"]) for s in scens],
                              env_trips=[s.n_trips for s in scens],
                              env_junctions=[len(s.graph["junc_lane_offsets"]) - 1 for s in scens]))
