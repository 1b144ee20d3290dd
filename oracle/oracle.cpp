// oracle.cpp — TEST INFRASTRUCTURE ONLY (see oracle.h header).
//
// A plain, serial, fp64 implementation of one simulation step of the model in
// DESIGN.md §1, written for reading against the paper:
//   * two-phase read/write separation: every decision reads state(t) only,
//     all writes are applied afterwards (§3.1 "Two-phase Parallel
//     Process for Read/Write Separation");
//   * per-lane order = the paper's linked list, here a std::vector sorted by
//     (s, vid) each step (§3.1 "Linked-list based Vehicle Sensing");
//   * IDM, randomized MOBIL, signal response,
//     App. A2.3;
//   * the Step() sequence of App. A2.2;
//   * signal policies incl. MAX_PRESSURE (
//     Varaiya 2013, readings L38-L41), metrics.
// Build: g++ -std=c++17 -O2 -ffp-contract=off -fno-fast-math -shared -fPIC.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

enum { PENDING = 0, DRIVING = 1, FINISHED = 2 };
enum { TURN_STRAIGHT = 0, TURN_LEFT = 1, TURN_RIGHT = 2 };
enum { KIND_NORMAL = 0, KIND_DYNAMIC = 1, KIND_TIDAL = 2 };
enum { POL_NONE = 0, POL_FIXED = 1, POL_MANUAL = 2, POL_MAXP = 3 };
enum { SIG_GREEN = 0, SIG_YELLOW = 1, SIG_RED = 2 };
const int LANE_DEST = -2, LANE_BLOCKED = -3;

struct Profile { double a_max, a_comf, T, s0, v_max, len; };

struct Vehicle {
  // static trip data
  int depart = 0, start_lane = 0, profile = 0;
  double start_s = 0, start_v = 0, end_s = 0;
  std::vector<int> route;
  bool on_net0 = false;
  // dynamic state
  int status = PENDING, lane = -1, cursor = 0, wait = 0;
  int insert_time = -1, arrive_time = -1;
  double s = 0, v = 0;
};

struct Junction {
  int policy = POL_NONE, phase = 0, elapsed = 0, yellow = 0, pending = 0;
  int request = -1;
  int pol_request = -1;                   // set_tl_policy, applied at the next step (L42)
  int remaining = -1;                     // MANUAL: green steps left in the current phase (L43)
  int dur_request = -1;                   // set_tl_duration, applied at the next step (L43)
  std::vector<int> lanes;                 // junction lanes (slot order)
  std::vector<std::vector<uint8_t>> green; // [phase][slot]
  std::vector<int> green_steps;
};

// The result of evaluating O4-O6 for a vehicle placed on a given lane.
struct LaneEval {
  double a = 0;
  bool has_leader = false;
  int leader = -1, hops = -1;
  double gap = 0, v_lead = 0;
  bool phantom = false;
  bool has_lim = false;
  double lim = 0, vlim = 0;
  int next1 = LANE_DEST;
};

struct Sim {
  // graph
  int nl = 0, nr = 0, nj = 0;
  std::vector<double> L, vmax;
  std::vector<int> road, junc, left, right, turn, kind, partner;
  std::vector<std::vector<int>> succ, pred, road_lanes;
  std::vector<int> lane_pos;               // index within its road (leftmost 0)
  std::vector<Junction> J;
  std::vector<int> lane_junc_slot;          // slot of a junction lane in its junction
  // params
  uint64_t seed = 0;
  std::vector<Profile> prof;
  double p_polite = 0.1, b_hard = 8, b_safe = 4, v_wait = 0.1, queue_zone = 100;
  int Y = 3, K = 2;
  int mp_period = 30;                      // MAX_PRESSURE decision period (L41)
  std::vector<uint8_t> restricted;         // set_lane_restriction flags (L44)
  bool store_fp32 = false, reverse_order = false;
  double start_margin = 0;
  // state
  int t = 0;
  std::vector<Vehicle> V;
  std::vector<int> dir;                     // lane direction flags
  std::vector<uint8_t> sig;                 // sig_t per lane (junction lanes)
  std::vector<std::vector<int>> pend;       // per lane pending vids by (depart, vid)
  std::vector<size_t> pend_head;
  // metrics
  int64_t vehicle_steps = 0, n_finished = 0, sum_travel = 0, sum_wait_fin = 0;
  int64_t sum_delay = 0, n_lc = 0, n_handoff = 0, n_inserted = 0;
  // decisions of the last step
  std::vector<int> d_leader, d_of, d_side;
  std::vector<int8_t> d_hops, d_phantom, d_lc, d_hand, d_fin, d_ins;
  std::vector<double> d_acc;

  bool is_road(int l) const { return road[l] >= 0; }
  bool is_lane(int m) const { return m >= 0; }
  int target_road(int j) const { return is_road(j) ? road[j] : road[succ[j][0]]; }

  // §1.3 usable(ℓ) (ledger L29, L30)
  bool usable(int l) const {
    if (restricted[l]) return false;                        // set_lane_restriction (L44)
    if (is_road(l)) return !(kind[l] == KIND_TIDAL && dir[l] != 0);
    int a = pred[l][0], b = succ[l][0];
    if (!usable(b)) return false;
    if (kind[a] != KIND_DYNAMIC) return true;
    if (turn[l] == TURN_LEFT) return dir[a] == 1;
    if (turn[l] == TURN_STRAIGHT) return dir[a] == 0;
    return true;
  }
  // §1.3 cand(ℓ, R'): lowest usable successor toward road R' (ledger L24)
  int min_cand(int l, int next_road) const {
    int best = LANE_BLOCKED;
    for (int j : succ[l])
      if (usable(j) && target_road(j) == next_road && (best < 0 || j < best)) best = j;
    return best;
  }
  // next lane from road lane l whose route index is ri (DEST on the last road).
  // Junction-lane choice (ledger L24): among usable successors toward
  // route[ri+1], the lowest id whose exit lane lies in the lane group toward
  // route[ri+2] (any lane on the destination road); if none, the lowest id.
  int next_from_road(int l, const Vehicle &k, int ri) const {
    if (ri + 1 >= (int)k.route.size()) return LANE_DEST;
    int R1 = k.route[ri + 1];
    int best_any = LANE_BLOCKED, best_pref = LANE_BLOCKED;
    for (int j : succ[l]) {
      if (!usable(j) || target_road(j) != R1) continue;
      if (best_any < 0 || j < best_any) best_any = j;
      int b = is_road(j) ? j : succ[j][0];
      bool pref = (ri + 2 >= (int)k.route.size()) || min_cand(b, k.route[ri + 2]) >= 0;
      if (pref && (best_pref < 0 || j < best_pref)) best_pref = j;
    }
    return best_pref >= 0 ? best_pref : best_any;
  }
  // next1 for vehicle k on lane l with cursor c (§1.3)
  int next1(int l, const Vehicle &k, int c) const {
    if (!is_road(l)) return succ[l][0];
    return next_from_road(l, k, c);
  }
  bool in_group(int a, const Vehicle &k, int c) const {   // lane group G
    if (c + 1 >= (int)k.route.size()) return true;
    return min_cand(a, k.route[c + 1]) >= 0;
  }

  // ---- IDM, P:158-161 with δ = 4; canonical order DESIGN §1.7 ----
  double idm(double v, double v0, bool has_leader, double gap, double dv,
             const Profile &p) const {
    double x = v / v0;
    double x2 = x * x;
    double x4 = x2 * x2;
    double fr = 1.0 - x4;
    double a;
    if (!has_leader) {
      a = p.a_max * fr;                                   // L7: no interaction term
    } else if (gap <= 0.0) {
      a = -b_hard;                                        // L8
    } else {
      double inv = 1.0 / (2.0 * std::sqrt(p.a_max * p.a_comf));
      double z = (v * p.T) + ((v * dv) * inv);
      double ss = p.s0 + std::max(0.0, z);
      double q = ss / gap;
      a = p.a_max * (fr - (q * q));
    }
    return std::max(a, -b_hard);
  }

  double veh_len(int vid) const { return prof[V[vid].profile].len; }
  double v0_of(int vid, int l) const { return std::min(vmax[l], prof[V[vid].profile].v_max); }

  // ---- O4-O6 for vehicle k placed on lane l at its own s, v (App. A2.3) ----
  // `lead_in_lane` is the in-lane leader (index into snapshot vid space) or -1.
  LaneEval eval_lane(int k, int l, int lead_in_lane,
                     const std::vector<std::vector<int>> &order) const {
    const Vehicle &me = V[k];
    const Profile &p = prof[me.profile];
    LaneEval e;
    e.next1 = next1(l, me, me.cursor);
    double v0 = v0_of(k, l);
    if (lead_in_lane >= 0) {                              // main pointer
      const Vehicle &f = V[lead_in_lane];
      e.has_leader = true; e.leader = lead_in_lane; e.hops = 0;
      e.gap = (f.s - me.s) - veh_len(lead_in_lane);
      e.v_lead = f.v;
    } else {                                              // P:168-169 substitution
      double d = L[l] - me.s;
      int m = e.next1;
      int ri = me.cursor;                                 // route index of last road lane
      for (int h = 1; h <= K; ++h) {
        if (!is_lane(m)) break;
        if (is_road(m)) ri += 1;
        if (!order[m].empty()) {
          int f = order[m][0];
          e.has_leader = true; e.leader = f; e.hops = h;
          e.gap = (d + V[f].s) - veh_len(f);
          e.v_lead = V[f].v;
          break;
        }
        d = d + L[m];
        m = is_road(m) ? next_from_road(m, me, ri) : succ[m][0];
      }
    }
    double a_lead = idm(me.v, v0, e.has_leader, e.gap, me.v - e.v_lead, p);
    e.a = a_lead;
    // O5 phantom: road lane, not destination road
    if (is_road(l) && e.next1 != LANE_DEST &&
        (e.next1 == LANE_BLOCKED || (!is_road(e.next1) && sig[e.next1] != SIG_GREEN))) {
      e.phantom = true;
      double gp = L[l] - me.s;
      double a_ph = idm(me.v, v0, true, gp, me.v - 0.0, p);
      e.a = std::min(a_lead, a_ph);
    }
    double lim_lead = me.s + e.gap;
    if (e.phantom && (!e.has_leader || L[l] <= lim_lead)) {
      e.has_lim = true; e.lim = L[l]; e.vlim = 0.0;
    } else if (e.has_leader) {
      e.has_lim = true; e.lim = lim_lead; e.vlim = e.v_lead;
    }
    return e;
  }

  // ---- signals (a5) ----
  void apply_requests() {
    // set_tl_policy (L42): the new policy from this step on; a
    // FIXED_TIME / MAX_PRESSURE junction restarts the current phase's green
    // timer (a running yellow completes); then phase requests (MANUAL)
    for (auto &j : J) {
      if (j.pol_request < 0) continue;
      const int np = j.pol_request;
      j.pol_request = -1;
      if (j.green.empty() || np == j.policy) continue;
      j.policy = np;
      if (np == POL_FIXED || np == POL_MAXP) j.elapsed = 0;
    }
    for (auto &j : J) {
      if (j.request >= 0) {
        int r = j.request;
        j.request = -1;
        j.policy = POL_MANUAL;
        j.remaining = -1;
        if (j.yellow > 0) {
          j.pending = r;
        } else if (r != j.phase) {
          if (Y > 0) { j.yellow = Y; j.pending = r; }
          else { j.phase = r; j.pending = r; }
        }
      }
      // set_tl_duration (L43): MANUAL, the (next) green is held for d steps
      if (j.dur_request >= 1 && !j.green.empty()) {
        j.policy = POL_MANUAL;
        j.remaining = j.dur_request;
      }
      j.dur_request = -1;
    }
  }
  void compute_signals() {
    for (auto &j : J) {
      for (size_t k = 0; k < j.lanes.size(); ++k) {
        int l = j.lanes[k];
        if (j.policy == POL_NONE || j.green.empty()) { sig[l] = SIG_GREEN; continue; }
        bool g = j.green[j.phase][k] != 0;
        if (j.yellow > 0) sig[l] = g ? SIG_YELLOW : SIG_RED;
        else sig[l] = g ? SIG_GREEN : SIG_RED;
      }
    }
  }
  // Max-pressure phase choice ("the junctions collect the pressures of
  // entering and exiting lanes and update the signal phases using the maximum
  // pressure algorithm"; Varaiya 2013): movement pressure of junction lane l =
  // count(predecessor lane) - count(successor lane) with counts = DRIVING
  // vehicles per lane in state(t) (L39); phase pressure = sum over its green
  // movements (L40); the argmax phase, ties -> lowest index.
  int max_pressure_phase(const Junction &j, const std::vector<std::vector<int>> &order) const {
    int best = 0;
    long long best_p = 0;
    for (size_t k = 0; k < j.green.size(); ++k) {
      long long pk = 0;
      for (size_t q = 0; q < j.lanes.size(); ++q) {
        if (!j.green[k][q]) continue;
        const int l = j.lanes[q];
        pk += (long long)order[pred[l][0]].size() - (long long)order[succ[l][0]].size();
      }
      if (k == 0 || pk > best_p) { best = (int)k; best_p = pk; }
    }
    return best;
  }
  // O11 for one junction; `order` = the lane order of state(t) (MAX_PRESSURE)
  void advance_junction(Junction &j, const std::vector<std::vector<int>> *order = nullptr) const {
    if (j.policy == POL_MAXP) {                  // L41
      if (j.yellow > 0) {
        j.yellow -= 1;
        if (j.yellow == 0) { j.phase = j.pending; j.elapsed = 0; }
      } else {
        j.elapsed += 1;
        if (j.elapsed >= mp_period) {
          const int nxt = max_pressure_phase(j, *order);
          if (nxt == j.phase) j.elapsed = 0;     // keep the green for another period
          else if (Y > 0) { j.yellow = Y; j.pending = nxt; }
          else { j.phase = nxt; j.pending = nxt; j.elapsed = 0; }
        }
      }
    } else if (j.policy == POL_FIXED) {
      if (j.yellow > 0) {
        j.yellow -= 1;
        if (j.yellow == 0) { j.phase = j.pending; j.elapsed = 0; }
      } else {
        j.elapsed += 1;
        if (!j.green_steps.empty() && j.elapsed >= j.green_steps[j.phase]) {
          int nxt = (j.phase + 1) % (int)j.green_steps.size();
          if (Y > 0) { j.yellow = Y; j.pending = nxt; }
          else { j.phase = nxt; j.pending = nxt; j.elapsed = 0; }
        }
      }
    } else if (j.policy == POL_MANUAL) {
      if (j.yellow > 0) {
        j.yellow -= 1;
        if (j.yellow == 0) j.phase = j.pending;
      } else if (j.remaining > 0) {              // L43: hold d green steps, then the next phase
        j.remaining -= 1;
        if (j.remaining == 0) {
          const int nxt = (j.phase + 1) % (int)j.green.size();
          if (Y > 0) { j.yellow = Y; j.pending = nxt; }
          else { j.phase = nxt; j.pending = nxt; }
          j.remaining = -1;
        }
      }
      j.elapsed += 1;
    }
  }

  // ---- lane order (O2, ties L12) ----
  std::vector<std::vector<int>> build_order() const {
    std::vector<std::vector<int>> order(nl);
    for (int k = 0; k < (int)V.size(); ++k)
      if (V[k].status == DRIVING) order[V[k].lane].push_back(k);
    for (auto &o : order)
      std::sort(o.begin(), o.end(), [&](int a, int b) {
        if (V[a].s != V[b].s) return V[a].s < V[b].s;
        return a < b;
      });
    return order;
  }

  void rebuild_pending() {
    pend.assign(nl, {});
    pend_head.assign(nl, 0);
    for (int k = 0; k < (int)V.size(); ++k)
      if (V[k].status == PENDING) pend[V[k].start_lane].push_back(k);
    for (auto &q : pend)
      std::sort(q.begin(), q.end(), [&](int a, int b) {
        if (V[a].depart != V[b].depart) return V[a].depart < V[b].depart;
        return a < b;
      });
  }

  // Philox4x32-10 (Salmon et al., SC'11; Random123 constants) — ledger L16
  static void philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
      uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
      uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
      uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
      uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
      uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
      c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
      k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
  }
  static double u53(uint64_t seed, int vid, int tt) {
    uint32_t ctr[4] = {(uint32_t)vid, (uint32_t)tt, 0u, 0u};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t x[4];
    philox(ctr, key, x);
    uint64_t m = ((uint64_t)(x[0] >> 5) << 26) + (uint64_t)(x[1] >> 6);
    return (double)m * (1.0 / 9007199254740992.0);
  }
  // p_LC, P:188-194 (ledger L14, literal piecewise)
  static double p_lc(double uT) {
    if (uT >= 1.0) return 0.9;
    if (uT > 0.0) return (0.9 - 2e-8) * uT;
    return 2e-8;
  }

  // ---- one step t -> t+1 (App. A2.2 Step()) ----
  struct Upd {
    bool moved = false, finished = false;
    int lane = -1, cursor = 0, wait = 0, lc = 0, hand = 0;
    double s = 0, v = 0, a = 0;
  };

  void step() {
    const int N = (int)V.size();
    apply_requests();                                       // L35
    compute_signals();                                      // O1
    std::vector<std::vector<int>> order = build_order();    // O2
    std::vector<int> pos(N, -1);
    for (int l = 0; l < nl; ++l)
      for (size_t i = 0; i < order[l].size(); ++i) pos[order[l][i]] = (int)i;

    d_leader.assign(N, -1); d_of.assign(N, -1); d_side.assign(4 * (size_t)N, -1);
    d_hops.assign(N, -1); d_phantom.assign(N, 0); d_lc.assign(N, 0);
    d_hand.assign(N, 0); d_fin.assign(N, 0); d_ins.assign(N, 0); d_acc.assign(N, 0.0);

    std::vector<Upd> upd(N);
    for (int it = 0; it < N; ++it) {
      int k = reverse_order ? N - 1 - it : it;
      if (V[k].status != DRIVING) continue;
      upd[k] = update_vehicle(k, order, pos);
    }

    // O10 departures (K11) — against state(t)
    std::vector<int> inserted;
    for (int l = 0; l < nl; ++l) {
      if (pend_head[l] >= pend[l].size()) continue;
      int k = pend[l][pend_head[l]];
      if (V[k].depart > t) continue;
      if (!usable(l)) continue;
      if (insertion_ok(k, l, order[l])) { inserted.push_back(k); pend_head[l]++; }
    }

    // ---- write phase (runtime partition) ----
    for (int k = 0; k < N; ++k) {
      if (!upd[k].moved) continue;
      Vehicle &me = V[k];
      const Upd &u = upd[k];
      vehicle_steps += 1;
      n_lc += (u.lc != 0);
      n_handoff += u.hand;
      me.wait = u.wait;
      if (u.finished) {
        me.status = FINISHED;
        me.arrive_time = t + 1;
        n_finished += 1;
        sum_travel += me.arrive_time - me.insert_time;    // L27
        sum_wait_fin += me.wait;
        me.lane = -1;
      } else {
        me.lane = u.lane; me.s = u.s; me.v = u.v; me.cursor = u.cursor;
      }
    }
    for (int k : inserted) {
      Vehicle &me = V[k];
      me.status = DRIVING; me.lane = me.start_lane; me.s = me.start_s; me.v = 0.0;
      me.cursor = 0; me.wait = 0; me.insert_time = t + 1;
      n_inserted += 1;
      sum_delay += me.insert_time - me.depart;
      d_ins[k] = 1;
    }
    if (store_fp32)
      for (auto &me : V)
        if (me.status == DRIVING) { me.s = (double)(float)me.s; me.v = (double)(float)me.v; }
    for (auto &j : J) advance_junction(j, &order);         // O11 (counts of state(t))
    t += 1;
  }

  bool insertion_ok(int k, int l, const std::vector<int> &ord) const {
    // L25: nearest ahead (first with s > start_s), nearest behind (last with s <= start_s)
    const Vehicle &me = V[k];
    const Profile &p = prof[me.profile];
    int ahead = -1, behind = -1;
    for (int x : ord) {
      if (V[x].s > me.start_s) { ahead = x; break; }
      behind = x;
    }
    if (ahead >= 0 && !(((V[ahead].s - me.start_s) - veh_len(ahead)) >= p.s0)) return false;
    if (behind >= 0) {
      const Profile &pb = prof[V[behind].profile];
      double need = (V[behind].v + 0.5 * pb.a_max) + p.s0;
      if (!(((me.start_s - V[behind].s) - p.len) >= need)) return false;
    } else {
      if (!((me.start_s - p.len) >= start_margin)) return false;
    }
    return true;
  }

  Upd update_vehicle(int k, const std::vector<std::vector<int>> &order,
                     const std::vector<int> &pos) {
    const Vehicle &me = V[k];
    const Profile &p = prof[me.profile];
    const int l = me.lane;
    const std::vector<int> &ol = order[l];
    int i = pos[k];
    int lead = (i + 1 < (int)ol.size()) ? ol[i + 1] : -1;  // main pointers
    int of = (i > 0) ? ol[i - 1] : -1;
    LaneEval cur = eval_lane(k, l, lead, order);
    d_leader[k] = cur.leader; d_hops[k] = (int8_t)cur.hops; d_phantom[k] = cur.phantom;
    d_of[k] = of;

    LaneEval use = cur;
    int lc = 0;
    int new_lane = l;
    if (is_road(l)) {                                       // P:95 no LC in junctions
      bool dest = me.cursor + 1 >= (int)me.route.size();
      bool inG = dest || cur.next1 != LANE_BLOCKED;
      // mandatory side (L18, L37)
      int mand = 0;
      if (!inG) {
        const std::vector<int> &rl = road_lanes[road[l]];
        bool left_ok = false, right_ok = false;
        for (int a : rl) {
          if (!usable(a) || !in_group(a, me, me.cursor)) continue;
          if (lane_pos[a] < lane_pos[l]) left_ok = true;
          if (lane_pos[a] > lane_pos[l]) right_ok = true;
        }
        mand = left_ok ? -1 : (right_ok ? +1 : 0);
      }
      bool l19 = (L[l] - me.s) < (p.s0 + (me.v * p.T));   // ledger L19
      // side pointers: front = first with s > s_k; back = last with s <= s_k (L11)
      int side_lane[2] = {left[l], right[l]};
      int front[2] = {-1, -1}, back[2] = {-1, -1};
      for (int sd = 0; sd < 2; ++sd) {
        int ls = side_lane[sd];
        if (ls < 0) continue;
        for (int x : order[ls]) {
          if (V[x].s > me.s) { front[sd] = x; break; }
          back[sd] = x;
        }
        d_side[4 * (size_t)k + 2 * sd + 0] = front[sd];
        d_side[4 * (size_t)k + 2 * sd + 1] = back[sd];
      }
      bool consider = inG ? !l19 : (mand != 0);
      if (consider) {
        // old follower terms (L10)
        double a_of = 0, a_of_new = 0;
        if (of >= 0) {
          const Vehicle &o = V[of];
          const Profile &po = prof[o.profile];
          double v0o = v0_of(of, l);
          a_of = idm(o.v, v0o, true, (me.s - o.s) - p.len, o.v - me.v, po);
          if (lead >= 0)
            a_of_new = idm(o.v, v0o, true, (V[lead].s - o.s) - veh_len(lead),
                           o.v - V[lead].v, po);
          else
            a_of_new = idm(o.v, v0o, false, 0.0, 0.0, po);
        }
        bool adm[2] = {false, false};
        double u[2] = {0, 0};
        LaneEval ev[2];
        for (int sd = 0; sd < 2; ++sd) {
          int ls = side_lane[sd];
          int sgn = sd == 0 ? -1 : +1;
          if (ls < 0 || !usable(ls)) continue;
          if (inG && !in_group(ls, me, me.cursor)) continue;
          if (!inG && sgn != mand) continue;
          ev[sd] = eval_lane(k, ls, front[sd], order);
          double a_nf = 0, a_nf_new = 0;
          bool ok = true;
          if (back[sd] >= 0) {
            const Vehicle &b = V[back[sd]];
            const Profile &pb = prof[b.profile];
            double v0b = v0_of(back[sd], ls);
            if (front[sd] >= 0)
              a_nf = idm(b.v, v0b, true, (V[front[sd]].s - b.s) - veh_len(front[sd]),
                         b.v - V[front[sd]].v, pb);
            else
              a_nf = idm(b.v, v0b, false, 0.0, 0.0, pb);
            double gb = (me.s - b.s) - p.len;
            a_nf_new = idm(b.v, v0b, true, gb, b.v - me.v, pb);
            if (!(a_nf_new >= -b_safe)) ok = false;       // L17 (1)
            if (!(gb >= 0.0)) ok = false;                 // L17 (2)
          } else {
            if (!((me.s - p.len) >= start_margin)) ok = false;  // L17 (3)
          }
          if (front[sd] >= 0) {
            double gf = (V[front[sd]].s - me.s) - veh_len(front[sd]);
            if (!(gf >= 0.0)) ok = false;                 // L17 (2)
          }
          // MOBIL utility (tilde = after the change, L13)
          u[sd] = (ev[sd].a - cur.a) + p_polite * ((a_nf_new - a_nf) + (a_of_new - a_of));
          adm[sd] = ok;
        }
        int choice = -1;
        if (inG) {
          if (adm[0] || adm[1]) {
            double uT = (adm[0] ? std::max(0.0, u[0]) : 0.0) +
                        (adm[1] ? std::max(0.0, u[1]) : 0.0);
            double pl = p_lc(uT);
            double r = u53(seed, k, t);                        // L16
            if (r < pl) {
              if (adm[0] && adm[1]) choice = (u[0] >= u[1]) ? 0 : 1;
              else choice = adm[0] ? 0 : 1;
            }
          }
        } else {
          int sd = mand < 0 ? 0 : 1;
          if (adm[sd]) choice = sd;                            // L18
        }
        if (choice >= 0) {
          use = ev[choice];
          lc = choice == 0 ? -1 : +1;
          new_lane = side_lane[choice];
        }
      }
    }
    d_lc[k] = (int8_t)lc;
    d_acc[k] = use.a;

    // O8 integrate (ledger L1) + clamp (L22, L23)
    Upd u;
    u.moved = true;
    u.lc = lc;
    double a = use.a;
    double vr = me.v + a;
    double s1, v1;
    if (vr < 0.0) { s1 = me.s - ((me.v * me.v) / (2.0 * a)); v1 = 0.0; }
    else { s1 = me.s + ((me.v + vr) * 0.5); v1 = vr; }
    if (use.has_lim && s1 > use.lim) {
      if (use.lim < me.s) { s1 = me.s; v1 = 0.0; }
      else { s1 = use.lim; v1 = std::min(v1, use.vlim); }
    }
    // O9 hand-off / arrival (L26, L31)
    int curl = new_lane, ri = me.cursor, n = use.next1, hand = 0;
    bool fin = false;
    for (;;) {
      bool dest_road = is_road(curl) && ri + 1 >= (int)me.route.size();
      if (dest_road && s1 >= me.end_s) { fin = true; break; }
      if (s1 > L[curl] && is_lane(n)) {
        s1 = s1 - L[curl];
        curl = n;
        if (is_road(curl)) ri += 1;
        hand += 1;
        n = is_road(curl) ? next_from_road(curl, me, ri) : succ[curl][0];
        continue;
      }
      break;
    }
    u.finished = fin;
    u.lane = curl; u.cursor = ri; u.s = s1; u.v = v1; u.hand = hand; u.a = a;
    u.wait = me.wait + ((v1 < v_wait) ? 1 : 0);            // L28
    d_hand[k] = (int8_t)std::min(hand, 127);
    d_fin[k] = fin;
    return u;
  }
};

std::string g_last_err;

}  // namespace

extern "C" {

void *or_create(const or_graph *g, const or_trips *tr, const or_params *pp,
                char *err, int32_t errlen) {
  auto fail = [&](const std::string &m) -> void * {
    if (err && errlen > 0) { std::snprintf(err, (size_t)errlen, "%s", m.c_str()); }
    return nullptr;
  };
  Sim *S = new Sim();
  S->nl = g->n_lanes; S->nr = g->n_roads; S->nj = g->n_junctions;
  int nl = S->nl;
  S->L.resize(nl); S->vmax.resize(nl); S->road.resize(nl); S->junc.resize(nl);
  S->left.resize(nl); S->right.resize(nl); S->turn.resize(nl); S->kind.resize(nl);
  S->partner.resize(nl); S->succ.assign(nl, {}); S->pred.assign(nl, {});
  S->restricted.assign(nl, 0);
  S->dir.resize(nl); S->sig.assign(nl, SIG_GREEN); S->lane_pos.assign(nl, 0);
  S->lane_junc_slot.assign(nl, -1);
  for (int l = 0; l < nl; ++l) {
    S->L[l] = (double)g->lane_length[l];
    S->vmax[l] = (double)g->lane_max_speed[l];
    S->road[l] = g->lane_road[l]; S->junc[l] = g->lane_junction[l];
    S->left[l] = g->lane_left[l]; S->right[l] = g->lane_right[l];
    S->turn[l] = g->lane_turn[l]; S->kind[l] = g->lane_kind[l];
    S->partner[l] = g->tidal_partner[l]; S->dir[l] = g->lane_dir0[l];
    for (int e = g->succ_offsets[l]; e < g->succ_offsets[l + 1]; ++e) {
      S->succ[l].push_back(g->succ_lanes[e]);
      S->pred[g->succ_lanes[e]].push_back(l);
    }
  }
  for (int l = 0; l < nl; ++l)
    if (!S->is_road(l) && (S->succ[l].size() != 1 || S->pred[l].size() != 1)) {
      delete S; return fail("junction lane " + std::to_string(l) + " needs one predecessor and one successor");
    }
  S->road_lanes.assign(S->nr, {});
  for (int r = 0; r < S->nr; ++r)
    for (int e = g->road_lane_offsets[r]; e < g->road_lane_offsets[r + 1]; ++e) {
      int l = g->road_lanes[e];
      S->lane_pos[l] = (int)S->road_lanes[r].size();
      S->road_lanes[r].push_back(l);
    }
  S->J.assign(S->nj, Junction());
  int64_t gidx = 0;
  for (int j = 0; j < S->nj; ++j) {
    Junction &J = S->J[j];
    for (int e = g->junc_lane_offsets[j]; e < g->junc_lane_offsets[j + 1]; ++e) {
      S->lane_junc_slot[g->junc_lanes[e]] = (int)J.lanes.size();
      J.lanes.push_back(g->junc_lanes[e]);
    }
    int np = g->junc_phase_offsets[j + 1] - g->junc_phase_offsets[j];
    for (int k = 0; k < np; ++k) {
      J.green.emplace_back(J.lanes.size());
      for (size_t s = 0; s < J.lanes.size(); ++s) J.green.back()[s] = g->phase_green[gidx++];
      J.green_steps.push_back(g->phase_green_steps[g->junc_phase_offsets[j] + k]);
    }
    J.policy = g->junc_policy[j];
    if (np == 0 && J.policy != POL_NONE) J.policy = POL_NONE;
  }
  // params
  S->seed = pp->seed;
  for (int i = 0; i < pp->n_profiles; ++i) {
    const float *r = pp->profiles + 6 * i;
    S->prof.push_back({(double)r[0], (double)r[1], (double)r[2], (double)r[3],
                       (double)r[4], (double)r[5]});
  }
  S->p_polite = (double)pp->politeness; S->b_hard = (double)pp->b_hard;
  S->b_safe = (double)pp->b_safe; S->v_wait = (double)pp->v_wait;
  S->queue_zone = (double)pp->queue_zone_m;
  S->Y = pp->yellow_steps; S->K = pp->lookahead_lanes;
  S->mp_period = pp->max_pressure_period > 0 ? pp->max_pressure_period : 30;
  S->store_fp32 = pp->store_fp32 != 0; S->reverse_order = pp->reverse_order != 0;
  // lane-start margin (L17): v_cap + 0.5 * a_cap, from the fp32 inputs
  double vcap = 0, acap = 0;
  for (int l = 0; l < nl; ++l) vcap = std::max(vcap, S->vmax[l]);
  for (auto &pr : S->prof) acap = std::max(acap, pr.a_max);
  S->start_margin = vcap + 0.5 * acap;
  // initial signal state: FIXED_TIME advanced offset steps
  for (int j = 0; j < S->nj; ++j) {
    Junction &J = S->J[j];
    if (J.policy == POL_FIXED) {
      int pol = J.policy;
      for (int s = 0; s < g->junc_offset_steps[j]; ++s) S->advance_junction(J);
      J.policy = pol;
    }
  }
  // trips
  S->V.resize(tr->n_trips);
  for (int k = 0; k < tr->n_trips; ++k) {
    Vehicle &v = S->V[k];
    v.depart = tr->depart_step[k];
    v.start_lane = tr->start_lane[k];
    v.start_s = (double)tr->start_s[k]; v.start_v = (double)tr->start_v[k];
    v.end_s = (double)tr->end_s[k]; v.profile = tr->profile[k];
    for (int e = tr->route_offsets[k]; e < tr->route_offsets[k + 1]; ++e)
      v.route.push_back(tr->route_roads[e]);
    if (v.route.empty()) { delete S; return fail("empty route for trip " + std::to_string(k)); }
    if (v.profile >= (int)S->prof.size()) { delete S; return fail("bad profile"); }
    v.on_net0 = tr->on_network_at_t0[k] != 0;
    if (v.on_net0) {
      v.status = DRIVING; v.lane = v.start_lane; v.s = v.start_s; v.v = v.start_v;
      v.cursor = 0; v.insert_time = 0;
    }
  }
  S->rebuild_pending();
  return S;
}

void or_destroy(void *h) { delete (Sim *)h; }

int32_t or_step(void *h, int32_t n) {
  Sim *S = (Sim *)h;
  for (int i = 0; i < n; ++i) S->step();
  return 0;
}

void or_read_state(void *h, or_state *o) {
  Sim *S = (Sim *)h;
  o->t = S->t;
  for (size_t k = 0; k < S->V.size(); ++k) {
    const Vehicle &v = S->V[k];
    o->status[k] = (uint8_t)v.status;
    o->lane[k] = v.status == DRIVING ? v.lane : -1;
    o->cursor[k] = v.status == DRIVING ? v.cursor : 0; o->wait_steps[k] = v.wait;
    o->insert_time[k] = v.insert_time; o->arrive_time[k] = v.arrive_time;
    o->s[k] = v.s; o->v[k] = v.v;
  }
  for (int j = 0; j < S->nj; ++j) {
    const Junction &J = S->J[j];
    o->junc_policy[j] = (uint8_t)J.policy; o->junc_phase[j] = J.phase;
    o->junc_elapsed[j] = J.elapsed; o->junc_yellow_left[j] = J.yellow;
    o->junc_pending[j] = J.pending;
    o->junc_remaining[j] = J.remaining;
  }
  for (int l = 0; l < S->nl; ++l) { o->lane_dir[l] = (uint8_t)S->dir[l]; o->lane_signal[l] = S->sig[l]; }
}

void or_load_state(void *h, const or_state *in) {
  Sim *S = (Sim *)h;
  S->t = in->t;
  for (size_t k = 0; k < S->V.size(); ++k) {
    Vehicle &v = S->V[k];
    v.status = in->status[k]; v.lane = in->lane[k]; v.cursor = in->cursor[k];
    v.wait = in->wait_steps[k]; v.insert_time = in->insert_time[k];
    v.arrive_time = in->arrive_time[k]; v.s = in->s[k]; v.v = in->v[k];
  }
  for (int j = 0; j < S->nj; ++j) {
    Junction &J = S->J[j];
    J.policy = in->junc_policy[j]; J.phase = in->junc_phase[j];
    J.elapsed = in->junc_elapsed[j]; J.yellow = in->junc_yellow_left[j];
    J.pending = in->junc_pending[j]; J.request = -1;
    J.remaining = in->junc_remaining[j]; J.pol_request = -1; J.dur_request = -1;
  }
  for (int l = 0; l < S->nl; ++l) S->dir[l] = in->lane_dir[l];
  S->rebuild_pending();
}

void or_lane_order(void *h, int32_t *offsets, int32_t *vids) {
  Sim *S = (Sim *)h;
  auto order = S->build_order();
  int32_t off = 0;
  for (int l = 0; l < S->nl; ++l) {
    offsets[l] = off;
    for (int k : order[l]) vids[off++] = k;
  }
  offsets[S->nl] = off;
}

void or_read_decisions(void *h, or_decisions *o) {
  Sim *S = (Sim *)h;
  size_t N = S->V.size();
  if (S->d_leader.size() != N) return;
  for (size_t k = 0; k < N; ++k) {
    o->leader_vid[k] = S->d_leader[k]; o->leader_hops[k] = S->d_hops[k];
    o->phantom[k] = S->d_phantom[k]; o->old_follower_vid[k] = S->d_of[k];
    for (int q = 0; q < 4; ++q) o->side_vid[4 * k + q] = S->d_side[4 * k + q];
    o->lc[k] = S->d_lc[k]; o->handoffs[k] = S->d_hand[k]; o->accel[k] = S->d_acc[k];
    o->finished[k] = S->d_fin[k]; o->inserted[k] = S->d_ins[k];
  }
}

void or_read_metrics(void *h, or_metrics *m) {
  Sim *S = (Sim *)h;
  m->t = S->t;
  int64_t pend = 0, drv = 0, fin = 0, tdrv = 0;
  for (auto &v : S->V) {
    pend += v.status == PENDING; drv += v.status == DRIVING; fin += v.status == FINISHED;
    if (v.status == DRIVING) tdrv += S->t - v.insert_time;   // time so far of a trip in progress
  }
  m->sum_time_driving = tdrv;
  m->n_pending = pend; m->n_driving = drv; m->n_finished = fin;
  m->vehicle_steps = S->vehicle_steps; m->sum_travel_steps = S->sum_travel;
  m->sum_wait_steps_finished = S->sum_wait_fin; m->sum_depart_delay = S->sum_delay;
  m->n_lane_changes = S->n_lc; m->n_handoffs = S->n_handoff; m->n_inserted = S->n_inserted;
}

void or_lane_stats(void *h, int32_t *cnt, int32_t *waiting) {
  // lane queue length: v < v_wait within the last queue_zone metres
  Sim *S = (Sim *)h;
  for (int l = 0; l < S->nl; ++l) { cnt[l] = 0; waiting[l] = 0; }
  for (auto &v : S->V) {
    if (v.status != DRIVING) continue;
    cnt[v.lane] += 1;
    if (v.v < S->v_wait && (S->L[v.lane] - v.s) <= S->queue_zone) waiting[v.lane] += 1;
  }
}

int32_t or_set_signal_phase(void *h, int32_t j, int32_t phase) {
  Sim *S = (Sim *)h;
  if (j < 0 || j >= S->nj) return 2;
  if (phase < 0 || phase >= (int)S->J[j].green.size()) return 2;
  S->J[j].request = phase;
  return 0;
}

int32_t or_set_signal_policy(void *h, int32_t j, int32_t policy) {
  Sim *S = (Sim *)h;
  if (j < 0 || j >= S->nj || policy < POL_NONE || policy > POL_MAXP) return 2;
  S->J[j].pol_request = policy;
  return 0;
}

int32_t or_set_vehicle_route(void *h, int32_t k, int32_t n, const int32_t *roads, float end_s) {
  // set_vehicle_route (L46): the remaining trip becomes roads[0..n),
  // starting with the current road (inside a junction also the committed next
  // road); the route cursor restarts at 0
  Sim *S = (Sim *)h;
  if (k < 0 || k >= (int)S->V.size() || n < 1) return 2;
  const int nr = (int)S->road_lanes.size();
  for (int e = 0; e < n; ++e) {
    if (roads[e] < 0 || roads[e] >= nr) return 2;
    if (e + 1 < n) {                                   // connected: some lane of roads[e] leads to roads[e+1]
      bool ok = false;
      for (int l : S->road_lanes[roads[e]])
        for (int j : S->succ[l]) ok |= S->target_road(j) == roads[e + 1];
      if (!ok) return 1;
    }
  }
  const int dl = S->road_lanes[roads[n - 1]][0];
  if (!((double)end_s >= 0.0 && (double)end_s <= S->L[dl])) return 1;
  Vehicle &v = S->V[k];
  if (v.status == FINISHED) return 1;
  if (v.status == DRIVING) {
    if (roads[0] != v.route[v.cursor]) return 1;
    if (!S->is_road(v.lane) && (n < 2 || (int)v.route.size() <= v.cursor + 1 || roads[1] != v.route[v.cursor + 1]))
      return 1;
  } else if (roads[0] != v.route[0]) {
    return 1;
  }
  v.route.assign(roads, roads + n);
  v.cursor = 0;
  v.end_s = (double)end_s;
  return 0;
}

int32_t or_set_signal_duration(void *h, int32_t j, int32_t steps) {
  Sim *S = (Sim *)h;
  if (j < 0 || j >= S->nj || steps < 1) return 2;
  S->J[j].dur_request = steps;
  return 0;
}

int32_t or_set_lane_max_speed(void *h, int32_t l, float v) {
  // set_lane_max_speed: v0 = min(lane, vehicle) from the next step (L6)
  Sim *S = (Sim *)h;
  if (l < 0 || l >= S->nl) return 2;
  if (!(v > 0.0f) || !std::isfinite(v)) return 1;
  S->vmax[l] = (double)v;
  return 0;
}

int32_t or_set_lane_restriction(void *h, int32_t l, int32_t flag) {
  // set_lane_restriction (L44): a restricted lane is not usable
  Sim *S = (Sim *)h;
  if (l < 0 || l >= S->nl || flag < 0 || flag > 1) return 2;
  S->restricted[l] = (uint8_t)flag;
  return 0;
}

void or_road_avg_speed(void *h, double *out) {
  // road travelling speed: mean speed of the vehicles on the
  // road's lanes; no vehicle -> free-flow speed = max lane speed of the road (L45)
  Sim *S = (Sim *)h;
  const int nr = (int)S->road_lanes.size();
  std::vector<double> sum(nr, 0.0);
  std::vector<long> cnt(nr, 0);
  for (auto &v : S->V) {
    if (v.status != DRIVING || !S->is_road(v.lane)) continue;
    sum[S->road[v.lane]] += v.v;
    cnt[S->road[v.lane]] += 1;
  }
  for (int r = 0; r < nr; ++r) {
    if (cnt[r]) { out[r] = sum[r] / (double)cnt[r]; continue; }
    double vm = 0.0;
    for (int l : S->road_lanes[r]) vm = std::max(vm, S->vmax[l]);
    out[r] = vm;
  }
}

int32_t or_set_lane_direction(void *h, int32_t l, int32_t d) {
  Sim *S = (Sim *)h;
  if (l < 0 || l >= S->nl || d < 0 || d > 1) return 2;
  if (S->kind[l] == KIND_DYNAMIC) { S->dir[l] = d; return 0; }
  if (S->kind[l] == KIND_TIDAL) {
    S->dir[l] = d;
    if (S->partner[l] >= 0) S->dir[S->partner[l]] = 1 - d;
    return 0;
  }
  return 1;
}

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  Sim::philox(ctr, key, out);
}
double or_u53(uint64_t seed, int32_t vid, int32_t t) { return Sim::u53(seed, vid, t); }

double or_idm(double v, double v0, int32_t has_leader, double gap, double dv,
              double a_max, double a_comf, double T, double s0, double b_hard) {
  Sim S;
  S.b_hard = b_hard;
  Profile p{a_max, a_comf, T, s0, 0.0, 0.0};
  return S.idm(v, v0, has_leader != 0, gap, dv, p);
}
double or_p_lc(double u) { return Sim::p_lc(u); }

}  // extern "C"
