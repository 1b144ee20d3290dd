// model.cuh — the per-vehicle model of DESIGN.md §1.5 (O4-O9), templated on
// the arithmetic type R:
//   * R = double: the canonical operation sequence of DESIGN §1.7 (each op a
//     separately rounded IEEE fp64 op via __dadd_rn/__dmul_rn/__ddiv_rn);
//     used by exact_mode and by the guard fallback;
//   * R = float: the fast path; every decision whose fp32 margin is inside the
//     guard band sets Guard::hit and the vehicle is recomputed with R = double.
// Paper: IDM P:156-167, randomized MOBIL P:171-198, signal P:200,
// substitution of the next lane's first vehicle P:168-169 (App. A2.3).
#pragma once
#include <math.h>
#include <stdint.h>

#include "dev.h"


namespace sim {

template <typename R> struct Ar;
template <> struct Ar<double> {
  static constexpr bool fp64 = true;
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double sub(double a, double b) { return __dadd_rn(a, -b); }
  __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <> struct Ar<float> {
  static constexpr bool fp64 = false;
  __device__ __forceinline__ static float add(float a, float b) { return a + b; }
  __device__ __forceinline__ static float sub(float a, float b) { return a - b; }
  __device__ __forceinline__ static float mul(float a, float b) { return a * b; }
  __device__ __forceinline__ static float div(float a, float b) { return __fdividef(a, b); }
};

// guard band of the fp32 path
constexpr float kEpsPos = 4e-6f;    // relative to the magnitude of the positions involved
constexpr float kEpsAcc = 2e-4f;    // m/s^2, accelerations / utilities
constexpr float kEpsP = 2e-4f;      // draw vs p_LC
constexpr float kEpsV = 2e-5f;      // relative, speed vs v_wait

struct Guard { bool hit; };

template <typename R> struct PV { R a_max, a_comf, T, s0, vmax, len, inv2; };
__device__ __forceinline__ PV<double> pvals(const Prof &p, double) {
  return {p.a_max_d, p.a_comf_d, p.T_d, p.s0_d, p.vmax_d, p.len_d, p.inv2sqrt_d};
}
__device__ __forceinline__ PV<float> pvals(const Prof &p, float) {
  return {p.a_max, p.a_comf, p.T, p.s0, p.vmax, p.len, p.inv2sqrt_f};
}

// IDM (delta = 4) in canonical order; ledger L7 (no leader), L8.
#ifdef KS_IDM_NOINLINE
#define IDM_INLINE __noinline__
#else
#define IDM_INLINE __forceinline__
#endif
template <typename R, bool GUARD>
__device__ IDM_INLINE R idm(R v, R v0, bool lead, R gap, R dv, const PV<R> &p, R b_hard,
                                 R gap_scale, Guard &g) {
  using M = Ar<R>;
  R x = M::div(v, v0);
  R x2 = M::mul(x, x);
  R x4 = M::mul(x2, x2);
  R fr = M::sub((R)1, x4);
  R a;
  if (!lead) {
    a = M::mul(p.a_max, fr);
  } else {
    if (GUARD && gap_scale > (R)0 && fabsf((float)gap) <= kEpsPos * (float)gap_scale) g.hit = true;
    if (gap <= (R)0) {
      a = -b_hard;
    } else {
      R z = M::add(M::mul(v, p.T), M::mul(M::mul(v, dv), p.inv2));
      R zz = ((R)0 < z) ? z : (R)0;
      R ss = M::add(p.s0, zz);
      R q = M::div(ss, gap);
      a = M::mul(p.a_max, M::sub(fr, M::mul(q, q)));
    }
  }
  return (a < -b_hard) ? -b_hard : a;
}

// usable successor of a tile road lane: j, its target road, exit lane b, the
// exit lane's reachable roads; fl: bit0 stop (junction lane not GREEN at t),
// bits 8-15 tile-local index of j when j is a junction lane of this tile
// (0xff: a direct road -> road link)
struct SuccEnt { int j, troad, b, fl; int4 outr; };

// Tile-local lane metadata staged in shared memory.
// the dynamic shared memory of k_step (StepSmem); tile tables inside a ring
// slot are addressed as offsets from it
extern __shared__ __align__(128) unsigned char ks_smem[];

struct TileSh {
  int nl, nroad, tile, base, ibase, cap, icap;
  int snap0, n;                      // snapshot range [snap0, snap0 + n) of the tile's vehicles
  int t;                             // the step (step_t(A), read once per tile)
  const Prof *P;                     // profile table (shared-memory copy when small)
  const ExtFirst *ext;               // [nl - nroad]: first vehicle of each junction lane's exit lane
  const PendHead *pend;              // [nroad]: heads of the pending-departure queues
  uint8_t sn[kMaxRoadLanes];         // usable successors per road lane
  uint8_t ng[kMaxRoadLanes];         // groups (distinct target roads) per road lane
  uint8_t gbeg[kMaxRoadLanes][kMaxGroups + 1];
  int gtroad[kMaxRoadLanes][kMaxGroups];
  // successor table and target-road section: read in place in the tile's
  // descriptor in the ring slot (byte offsets from ks_smem, so that every
  // access stays a shared-memory load); se0[l] = first entry of road lane l
  uint32_t se_o, tr_o;
  uint8_t se0[kMaxRoadLanes];
  int glob[kMaxTileLanes];
  float len[kMaxTileLanes], vmax[kMaxTileLanes];
  int16_t seg_start[kMaxTileLanes], seg_end[kMaxTileLanes];   // lane segments of the snapshot
  int first_out[kMaxTileLanes];      // (output rank << 15) | snapshot index of the lane's first stayer
  int8_t left[kMaxTileLanes], right[kMaxTileLanes];
  uint8_t isroad[kMaxTileLanes], usable[kMaxTileLanes];
  // the distinct roads the tile's road lanes lead to (<= 4 lanes x 4 groups):
  // reach[k] = road lanes with a usable successor toward troad[k],
  // gidx[a][k] = that group of lane a (-1 none); umask = usable road lanes.
  // A vehicle finds k for its next road once; every "lane a leads to my next
  // road" test is then one bit
  int ntr;
  uint32_t umask;
  // per-tile outputs of the step
  int run;                           // stayers written (compaction, in snapshot order)
  int c_fin, c_lc, c_hand, c_guard, c_ovf, c_ins;
  unsigned long long c_delay;
};

__device__ __forceinline__ const SuccEnt &t_se(const TileSh &T, int l, int k) {
  return reinterpret_cast<const SuccEnt *>(ks_smem + T.se_o)[T.se0[l] + k];
}
// target-road section: troad[32] (int), reach[32] (bytes), gidx[8][32] (bytes)
__device__ __forceinline__ int t_troad(const TileSh &T, int k) {
  return reinterpret_cast<const int *>(ks_smem + T.tr_o)[k];
}
__device__ __forceinline__ uint32_t t_reach(const TileSh &T, int k) {
  return (ks_smem + T.tr_o + 4 * kMaxRoadLanes * kMaxGroups)[k];
}
__device__ __forceinline__ int t_gidx(const TileSh &T, int l, int k) {
  return reinterpret_cast<const int8_t *>(ks_smem + T.tr_o + 5 * kMaxRoadLanes * kMaxGroups)
      [l * (kMaxRoadLanes * kMaxGroups) + k];
}

// Snapshot of a tile at time t (shared memory; the tile's global scratch for
// a tile in global mode): eight word arrays of stride st — the fields other
// vehicles read (s, v, vid, meta) and the fields only the vehicle itself uses
// (nxt, nxt2, wait, end_s), all merged once per step (a1).
struct View {
  uint32_t *p;
  int st;
  __device__ __forceinline__ float &s(int i) const { return reinterpret_cast<float *>(p)[i]; }
  __device__ __forceinline__ float &v(int i) const { return reinterpret_cast<float *>(p)[st + i]; }
  __device__ __forceinline__ int32_t &vid(int i) const { return reinterpret_cast<int32_t *>(p)[2 * st + i]; }
  __device__ __forceinline__ uint32_t &meta(int i) const { return p[3 * st + i]; }
  __device__ __forceinline__ int32_t &nxt(int i) const { return reinterpret_cast<int32_t *>(p)[4 * st + i]; }
  __device__ __forceinline__ int32_t &nxt2(int i) const { return reinterpret_cast<int32_t *>(p)[5 * st + i]; }
  __device__ __forceinline__ int32_t &wait(int i) const { return reinterpret_cast<int32_t *>(p)[6 * st + i]; }
  __device__ __forceinline__ float &ends(int i) const { return reinterpret_cast<float *>(p)[7 * st + i]; }
};

__device__ __forceinline__ int m_lane(uint32_t m) { return (int)(m & 0xffu); }
__device__ __forceinline__ int m_prof(uint32_t m) { return (int)((m >> 8) & 0xffu); }
__device__ __forceinline__ int m_cursor(uint32_t m) { return (int)(m >> 16); }

// route[idx] beyond the cached next two roads (rare: lookahead / hand-offs
// past the next road), out of line to keep the hot passes small
static __device__ __noinline__ int route_far(const StepArgs &A, int vid, int idx) {
  int off = __ldg(A.route_start + vid);
  int len = __ldg(A.route_len + vid);
  return (idx >= 0 && idx < len) ? __ldg(A.route + off + idx) : -1;
}
__device__ __forceinline__ int route_at(const StepArgs &A, int vid, int c, int nxt, int nxt2,
                                        int idx) {
  if (idx == c + 1) return nxt;
  if (idx == c + 2) return nxt2;
  return route_far(A, vid, idx);
}

__device__ __forceinline__ bool in4(const int4 &o, int R) {
  return o.x == R || o.y == R || o.z == R || o.w == R;
}

// cand(b, R) != empty, global lane b: the distinct roads
// reachable through usable successors (<= 4 per lane, validated at create)
__device__ __forceinline__ bool has_outroad(const StepArgs &A, int b, int R) {
  return in4(__ldg(A.outroads + b), R);
}
__device__ __forceinline__ bool pref_ok(const int4 &outr, int R2) {
  return R2 < 0 || in4(outr, R2);
}

// next lane from road lane m toward road R1 with preference toward R2 (ledger L24)
__device__ __forceinline__ int next_from_road(const StepArgs &A, int m, int R1, int R2) {
  if (R1 < 0) return kLaneDest;
  int best_any = kLaneBlocked, best_pref = kLaneBlocked;
  int e1 = __ldg(A.succ_off + m + 1);
#pragma unroll 1
  for (int e = __ldg(A.succ_off + m); e < e1; ++e) {
    int j = __ldg(A.succ + e);
    if (!A.usable[j] || __ldg(A.target_road + j) != R1) continue;
    if (best_any < 0 || j < best_any) best_any = j;
    const int b = __ldg(A.exit_lane + j);
    if (pref_ok(__ldg(A.outroads + b), R2) && (best_pref < 0 || j < best_pref)) best_pref = j;
  }
  return best_pref >= 0 ? best_pref : best_any;
}
// the same two predicates for a road lane of this tile, from the shared-memory
// successor table (built per step; usable successors only)
__device__ __forceinline__ bool has_outroad_t(const StepArgs &A, const TileSh &T, int a, int R) {
  for (int g = 0; g < T.ng[a]; ++g)
    if (T.gtroad[a][g] == R) return true;
  return false;
}
// next lane, "stop line applies" (junction lane not GREEN) and how to find
// the lane's first vehicle without a global lookup: hint >= 0 is the
// tile-local index of a junction lane of this tile (snapshot segment), -1
// none (generic lookup)
struct Next { int j; bool stop; int hint; };
__device__ __forceinline__ Next ent_next(const SuccEnt &x) {
  const int jl = (x.fl >> 8) & 0xff;
  return Next{x.j, (x.fl & 1) != 0, jl == 0xff ? -1 : jl};
}
__device__ __forceinline__ Next next1_t(const StepArgs &A, const TileSh &T, int l, int R1, int R2) {
  if (R1 < 0) return Next{kLaneDest, false, -1};
  for (int g = 0; g < T.ng[l]; ++g) {
    if (T.gtroad[l][g] != R1) continue;
    const int b = T.gbeg[l][g], e = T.gbeg[l][g + 1];
    // entries sorted by lane id: the first is the lowest candidate, the first
    // whose exit lane continues toward R2 is the preferred one (ledger L24)
    for (int k = b; k < e; ++k) {
      const SuccEnt &x = t_se(T, l, k);
      if (pref_ok(x.outr, R2)) return ent_next(x);
    }
    return ent_next(t_se(T, l, b));
  }
  return Next{kLaneBlocked, false, -1};
}
// next1_t for the vehicle's own next road, known as troad[k] (k < 0: no road
// lane of the tile leads there)
__device__ __forceinline__ Next next1_k(const TileSh &T, int l, int k, int R2) {
  const int g = k >= 0 ? t_gidx(T, l, k) : -1;
  if (g < 0) return Next{kLaneBlocked, false, -1};
  const int b = T.gbeg[l][g], e = T.gbeg[l][g + 1];
  for (int q = b; q < e; ++q) {
    const SuccEnt &x = t_se(T, l, q);
    if (pref_ok(x.outr, R2)) return ent_next(x);
  }
  return ent_next(t_se(T, l, b));
}
__device__ __forceinline__ int troad_index(const TileSh &T, int R) {
  for (int k = 0; k < T.ntr; ++k)
    if (t_troad(T, k) == R) return k;
  return -1;
}
__device__ __forceinline__ int next_from_road_t(const StepArgs &A, const TileSh &T, int l, int R1,
                                                int R2) {
  return next1_t(A, T, l, R1, R2).j;
}
// any road lane (global id g); out of line (hand-offs and deep lookahead only)
static __device__ __noinline__ int next_from_road_any(const StepArgs &A, const TileSh &T, int g,
                                                  int R1, int R2) {
  if (__ldg(A.lane_tile + g) == T.tile) {
    const int l = A.lane_local[g];
    if (l < T.nroad) return next_from_road_t(A, T, l, R1, R2);
  }
  return next_from_road(A, g, R1, R2);
}

struct First { bool found; float s, v, len; int vid; };

// direct transport: lane m of tile mt from its owner partition's buffers of t
// (out of line: keeps the single-partition lookahead path unchanged)
static __device__ __noinline__ unsigned long long peer_summary(const StepArgs &A, int mt, int m,
                                                        const float *&pv) {
  const PeerView &Q = A.peers[__ldg(A.tile_owner + mt)];
  pv = Q.pubv[step_t(A) & 1];
  return Q.summ[step_t(A) % 3][m];
}

// first vehicle of lane m at time t: from the tile snapshot if m is ours, else
// from the lane summary built race-free during step t-1
static __device__ __noinline__ First first_of(const StepArgs &A, const TileSh &T, const View &C, int m) {
  First f;
  f.found = false;
  const int mt = __ldg(A.lane_tile + m);
  if (mt == T.tile) {
    int ll = A.lane_local[m];
    int a = T.seg_start[ll];
    if (a < T.seg_end[ll]) {
      f.found = true;
      f.s = C.s(a);
      f.v = C.v(a);
      f.vid = C.vid(a);
      f.len = T.P[m_prof(C.meta(a))].len;
    }
  } else {
    // direct transport (NEXT-2): a lane of another partition is read from its
    // owner's summary of t, written there during step t-1 (no halo copy)
    unsigned long long key;
    const float *pv = A.pubv_cur;
    if (!A.peers) key = A.summ_cur[m];
    else key = peer_summary(A, mt, m, pv);
    if (key != kEmptyKey) {
      f.found = true;
      f.s = __uint_as_float((unsigned)(key >> 32));
      f.vid = (int)(unsigned)(key & 0xffffffffu);
      f.v = pv[f.vid];
      f.len = T.P[A.veh_prof[f.vid]].len;
    }
  }
  return f;
}
// first vehicle of the tile's own junction lane jl (snapshot segment)
__device__ __forceinline__ First first_local(const TileSh &T, const View &C, int jl) {
  First f;
  const int a = T.seg_start[jl];
  f.found = a < T.seg_end[jl];
  if (f.found) {
    f.s = C.s(a);
    f.v = C.v(a);
    f.vid = C.vid(a);
    f.len = T.P[m_prof(C.meta(a))].len;
  }
  return f;
}
__device__ __forceinline__ int xl_of(const TileSh &T, int jl) { return T.ext[jl - T.nroad].b; }
// first vehicle of the exit lane of the tile's junction lane jl (gathered)
__device__ __forceinline__ First first_ext(const TileSh &T, int jl) {
  const ExtFirst &x = T.ext[jl - T.nroad];
  First f;
  f.found = x.vid >= 0;
  f.s = x.s;
  f.v = x.v;
  f.vid = x.vid;
  f.len = x.len;
  return f;
}

template <typename R> struct LEv {
  R a, gap, vlead, lim, vlim;
  R limrel;                          // lim - s computed without cancellation (fp32 path)
  int leader, hops, next1;
  int nl1;                           // next1 as a junction lane of this tile (tile-local), else -1
  bool has_leader, phantom, has_lim;
};

struct Me {                          // the ego vehicle's identity / route cache
  int vid, cur, nxt, nxt2;
  float ends;                        // end position on the destination road
  int k;                             // index of nxt in the tile's target roads (TileSh::troad)
};

// O4-O6 for the ego placed on tile-local lane l (App. A2.3).
// The lookahead walks the next lanes along the route; the first
// two of them are resolved on chip in the common case — a junction lane of
// this tile (its snapshot segment) and that junction lane's exit lane (the
// first vehicle gathered by the producer warp) — and through the lane
// summaries otherwise (first_of).  The values read are the same either way.
template <typename R, bool GUARD>
__device__ __forceinline__ LEv<R> eval_lane(const StepArgs &A, const TileSh &T, const View &C, int l,
                                            int lead_idx, R s, R v, const PV<R> &p, const Me &me,
                                            Guard &g) {
  using M = Ar<R>;
  LEv<R> e;
  const bool road = T.isroad[l];
  Next nx;
  int ext = -1;                                          // junction lane whose exit lane is next
  if (road) {
    nx = me.nxt < 0 ? Next{kLaneDest, false, -1} : next1_k(T, l, me.k, me.nxt2);
  } else {                                               // junction lane: its exit lane
    nx = Next{xl_of(T, l), false, -1};
    ext = l;
  }
  e.next1 = nx.j;
  e.nl1 = road ? nx.hint : -1;
  const R vmax_l = (R)T.vmax[l];
  const R v0 = (p.vmax < vmax_l) ? p.vmax : vmax_l;
  const R L = (R)T.len[l];
  e.has_leader = false;
  e.leader = -1;
  e.hops = -1;
  e.gap = (R)0;
  e.vlead = (R)0;
  R gscale = (R)0;
  if (lead_idx >= 0) {                                   // main pointer
    R sf = (R)C.s(lead_idx);
    R lf = (R)T.P[m_prof(C.meta(lead_idx))].len;
    e.has_leader = true;
    e.leader = C.vid(lead_idx);
    e.hops = 0;
    e.gap = M::sub(M::sub(sf, s), lf);
    e.vlead = (R)C.v(lead_idx);
    gscale = fabs(sf - s) + lf;
  } else {                                               // P:168-169 substitution
    R d = M::sub(L, s);
    int m = e.next1, rel = 0;
    int own = road ? nx.hint : -1;                       // m is the tile's junction lane `own`
#pragma unroll 1
    for (int h = 1; h <= A.lookahead; ++h) {
      if (m < 0) break;
      First f;
      bool mroad;
      R Lm;
      if (own >= 0) {
        mroad = false;
        f = first_local(T, C, own);
        Lm = (R)T.len[own];
      } else if (ext >= 0) {
        mroad = true;                                    // exit lanes are road lanes
        f = first_ext(T, ext);
        Lm = (R)T.ext[ext - T.nroad].Lb;
      } else {
        mroad = __ldg(A.lane_road + m) >= 0;
        f = first_of(A, T, C, m);
        Lm = (R)__ldg(A.lane_len + m);
      }
      if (mroad) rel += 1;
      if (f.found) {
        e.has_leader = true;
        e.leader = f.vid;
        e.hops = h;
        e.gap = M::sub(M::add(d, (R)f.s), (R)f.len);
        e.vlead = (R)f.v;
        gscale = d + (R)f.s + (R)f.len;
        break;
      }
      d = M::add(d, Lm);
      if (!mroad) {
        if (own >= 0) { ext = own; m = xl_of(T, own); }
        else m = __ldg(A.exit_lane + m);
        own = -1;
      } else {
        ext = -1;
        own = -1;
        int R1 = route_at(A, me.vid, me.cur, me.nxt, me.nxt2, me.cur + rel + 1);
        int R2 = route_at(A, me.vid, me.cur, me.nxt, me.nxt2, me.cur + rel + 2);
        m = next_from_road_any(A, T, m, R1, R2);
      }
    }
  }
  const R b_hard = (R)A.b_hard;
  R a_lead = idm<R, GUARD>(v, v0, e.has_leader, e.gap, M::sub(v, e.vlead), p, b_hard, gscale, g);
  e.a = a_lead;
  e.phantom = false;
  if (road && e.next1 != kLaneDest && (e.next1 == kLaneBlocked || nx.stop)) {
    e.phantom = true;                                    // P:200 stationary vehicle at lane end
    R gp = M::sub(L, s);                                 // sign exact: no guard needed
    R a_ph = idm<R, GUARD>(v, v0, true, gp, M::sub(v, (R)0), p, b_hard, (R)0, g);
    e.a = (a_ph < a_lead) ? a_ph : a_lead;
  }
  R lim_lead = M::add(s, e.gap);
  e.has_lim = false;
  e.lim = (R)0;
  e.vlim = (R)0;
  e.limrel = (R)0;
  if (GUARD && e.phantom && e.has_leader &&
      fabsf((float)(L - lim_lead)) <= kEpsPos * (float)(L + fabs(lim_lead)))
    g.hit = true;
  if (e.phantom && (!e.has_leader || L <= lim_lead)) {
    e.has_lim = true;
    e.lim = L;
    e.limrel = M::sub(L, s);
    e.vlim = (R)0;
  } else if (e.has_leader) {
    e.has_lim = true;
    e.lim = lim_lead;
    e.limrel = e.gap;
    e.vlim = e.vlead;
  }
  return e;
}

struct Res {
  float s1, v1, acc;
  int nxt, nxt2;                     // route[c+1], route[c+2] of the snapshot (cursor c)
  int lane_g, cursor;
  int cl, cx;                        // lane_g as a lane of this tile (local index), else -1; if
                                     // lane_g is the exit lane of junction lane cx of this tile, cx
  int lc, hand;
  bool fin;
  int wait1;
};

__device__ __forceinline__ int upper_bound_s(const View &C, int a, int b, float s) {
  // first index in [a, b) with C.s > s   (side pointers; ties -> back, L11)
  while (a < b) {
    int mid = (a + b) >> 1;
    if (C.s(mid) > s) b = mid; else a = mid + 1;
  }
  return a;
}

template <typename R> struct SideRes {
  int choice;                        // -1 stay, 0 left, 1 right
  R a, lim, limrel, vlim;
  int next1, nl1;
  bool has_lim, hit;
};

// O7 decision for a vehicle with at least one admissible side:
// evaluates O4-O6 on the side lanes still able to win and picks the side.  On
// the fp32 path a side is evaluated only if the draw can still fall below
// p_LC: with F = the free-road IDM bound of ã_ego on that lane, u <= (F - a_cur)
// + p * pol, and p_LC is monotone in u_T apart from its 2e-8 floor, so r >=
// p_LC(upper bound) + 1e-3 decides "stay" exactly.  Out of line:
// it runs for ~1-2% of vehicles and keeps the hot loop small.
template <typename R, bool GUARD>
__device__ __noinline__ SideRes<R> lane_change(const StepArgs &A, const TileSh &T, const View &C,
                                               bool adm0, bool adm1, bool inG, int mand, int sl0,
                                               int sl1, int f0, int f1, R s, R v, const PV<R> p,
                                               const Me me, R a_cur, R pol0, R pol1, double r) {
  using M = Ar<R>;
  Guard g;
  g.hit = false;
  SideRes<R> o;
  o.choice = -1;
  bool need0 = adm0 && (inG || mand < 0);
  bool need1 = adm1 && (inG || mand > 0);
  const R b_hard = (R)A.b_hard;
  if (GUARD && inG && (need0 || need1)) {
    R ub = (R)0;
#pragma unroll 1
    for (int sd = 0; sd < 2; ++sd) {
      if (!(sd == 0 ? need0 : need1)) continue;
      const int ls = sd == 0 ? sl0 : sl1;
      const R v0s = (p.vmax < (R)T.vmax[ls]) ? p.vmax : (R)T.vmax[ls];
      const R x = M::div(v, v0s);
      const R x2 = M::mul(x, x);
      R F = M::mul(p.a_max, M::sub((R)1, M::mul(x2, x2)));
      F = (F < -b_hard) ? -b_hard : F;
      const R U = M::add(M::sub(F, a_cur), M::mul((R)A.polite, sd == 0 ? pol0 : pol1));
      ub = M::add(ub, ((R)0 < U) ? U : (R)0);
    }
    const double pmax = ub >= (R)1 ? 0.9 : fmax(2e-8, (double)(0.9 - 2e-8) * (double)ub);
    if (r >= pmax + 1e-3) need0 = need1 = false;       // no change, for certain
  }
  if (!(need0 || need1)) { o.hit = g.hit; return o; }
  // ã_ego on each side; keep the utility of both and the evaluation of the
  // side that would be taken (argmax, tie -> left: P:196, ledger L15)
  R u0 = (R)0, u1 = (R)0;
  LEv<R> best;
#pragma unroll 1
  for (int sd = 0; sd < 2; ++sd) {
    if (!(sd == 0 ? need0 : need1)) continue;
    const LEv<R> e = eval_lane<R, GUARD>(A, T, C, sd == 0 ? sl0 : sl1, sd == 0 ? f0 : f1, s, v, p,
                                         me, g);
    // MOBIL utility (tilde = after the change, ledger L13)
    const R u = M::add(M::sub(e.a, a_cur), M::mul((R)A.polite, sd == 0 ? pol0 : pol1));
    if (sd == 0) u0 = u; else u1 = u;
    if (sd == 0 || !need0 || u0 < u1) best = e;
  }
  int choice = -1;
  if (inG) {
    const R p0 = need0 ? (((R)0 < u0) ? u0 : (R)0) : (R)0;
    const R p1 = need1 ? (((R)0 < u1) ? u1 : (R)0) : (R)0;
    const R uT = M::add(p0, p1);
    double pl;                                           // P:188-194, ledger L14
    if (uT >= (R)1) pl = 0.9;
    else if (uT > (R)0) pl = (double)M::mul((R)(0.9 - 2e-8), uT);
    else pl = 2e-8;
    if (GUARD && fabs(r - pl) <= (double)kEpsP) g.hit = true;
    if (r < pl) {                                        // P:196, ledger L15
      if (need0 && need1) {
        if (GUARD && fabsf((float)(u0 - u1)) <= kEpsAcc) g.hit = true;
        choice = (u0 >= u1) ? 0 : 1;
      } else {
        choice = need0 ? 0 : 1;
      }
    }
  } else {
    choice = mand < 0 ? 0 : 1;                           // ledger L18: admissible -> change
  }
  o.choice = choice;
  o.a = best.a;
  o.lim = best.lim;
  o.limrel = best.limrel;
  o.vlim = best.vlim;
  o.next1 = best.next1;
  o.nl1 = best.nl1;
  o.has_lim = best.has_lim;
  o.hit = g.hit;
  return o;
}

// ---- one vehicle's update O4-O9, reading only state(t) ----
// Three pieces, so that the fp32 step kernel can run them as separate dense
// passes and the fp64 canonical path runs them back to back
// (veh_update): lc_elig + eval_lane (current lane), lc_decide (MOBIL, only
// for vehicles that may change lane), integrate (O8-O9).

struct Elig {                        // lane-change eligibility (L18, L19, L37)
  int sl0, sl1, mand;
  bool inG, want0, want1;
};

template <typename R, bool GUARD>
__device__ __forceinline__ Elig lc_elig(const StepArgs &A, const TileSh &T, int l, R s, R v,
                                        const PV<R> &p, Me &me, Guard &g) {
  using M = Ar<R>;
  Elig E;
  const R L = (R)T.len[l];
  bool inG = true, consider = false, want0 = false, want1 = false;
  int mand = 0, sl0 = -1, sl1 = -1;
  const bool dest = me.nxt < 0;
  me.k = -1;
  if (T.isroad[l]) {                                     // no LC in junction lanes
    // road lanes of the tile leading to the next road: one bit each
    uint32_t G = T.umask;                                // destination road: every usable lane
    if (!dest) {
      me.k = troad_index(T, me.nxt);
      G = me.k >= 0 ? t_reach(T, me.k) : 0u;
    }
    inG = dest || ((G >> l) & 1u);                       // l in G <=> next1 != BLOCKED
    if (!inG) {                                          // ledger L18, L37
      const uint32_t M = G & T.umask;
      mand = (M & ((1u << l) - 1u)) ? -1 : ((M >> (l + 1)) ? 1 : 0);
    }
    const R rem = M::sub(L, s);
    const R need = M::add(p.s0, M::mul(v, p.T));
    const bool l19 = rem < need;                         // ledger L19
    if (GUARD && inG && v != (R)0 && fabsf((float)(rem - need)) <= kEpsPos * (float)(fabs(rem) + need))
      g.hit = true;
    sl0 = T.left[l];
    sl1 = T.right[l];
    consider = inG ? !l19 : (mand != 0);
    if (consider) {
      // discretionary: usable side lanes that also lead to the next road;
      // mandatory (L18): the usable side lane toward G
      const uint32_t W = T.umask & (inG ? G : ~0u);
      want0 = sl0 >= 0 && ((W >> sl0) & 1u) && (inG || mand == -1);
      want1 = sl1 >= 0 && ((W >> sl1) & 1u) && (inG || mand == 1);
    }
  }
  E.sl0 = sl0;
  E.sl1 = sl1;
  E.mand = mand;
  E.inG = inG;
  E.want0 = want0;
  E.want1 = want1;
  return E;
}

// O7 for one vehicle: side pointers, admissibility,
// politeness, the draw and the decision (lane_change).  choice -1: stay.
template <typename R, bool GUARD>
__device__ __forceinline__ SideRes<R> lc_decide(const StepArgs &A, const TileSh &T, const View &C,
                                                int i, int l, R s, R v, const PV<R> &p, const Me &me,
                                                const Elig &E, R a_cur, Guard &g) {
  using M = Ar<R>;
  const R b_hard = (R)A.b_hard;
  const int sl0 = E.sl0, sl1 = E.sl1, mand = E.mand;
  const bool inG = E.inG, want0 = E.want0, want1 = E.want1;
  const int lead = (i + 1 < T.seg_end[l]) ? i + 1 : -1;
  const int of = (i > T.seg_start[l]) ? i - 1 : -1;
  int f0 = -1, f1 = -1, b0 = -1, b1 = -1;
#pragma unroll 1
  for (int sd = 0; sd < 2; ++sd) {                       // side pointers (ties -> back, L11)
    const int ls = sd == 0 ? sl0 : sl1;
    if (ls < 0 || !((sd == 0 ? want0 : want1) || A.record)) continue;
    const int a = T.seg_start[ls], b = T.seg_end[ls];
    const int f = upper_bound_s(C, a, b, C.s(i));
    const int fr = f < b ? f : -1, bk = f > a ? f - 1 : -1;
    if (sd == 0) { f0 = fr; b0 = bk; } else { f1 = fr; b1 = bk; }
    if (A.record) {
      A.r_side[4 * me.vid + 2 * sd] = fr >= 0 ? C.vid(fr) : -1;
      A.r_side[4 * me.vid + 2 * sd + 1] = bk >= 0 ? C.vid(bk) : -1;
    }
  }
  // ---- MOBIL admissibility of each side, cheapest test first (gap signs,
  // lane-start rule, then the b_safe IDM of the new follower); the politeness
  // terms (L10, L13, L17) only for admissible sides.  A test that
  // fails outside its guard band decides "inadmissible" exactly, so the later
  // ones are skipped ----
  bool adm0 = false, adm1 = false;
  R pol0 = (R)0, pol1 = (R)0;                            // (ã_nf - a_nf) + (ã_of - a_of)
  double r = 1.0;                                        // U53 draw (L16), discretionary only
  if (want0 || want1) {
    R anew0 = (R)0, anew1 = (R)0;                        // ã_nf per side
#pragma unroll 1
    for (int sd = 0; sd < 2; ++sd) {
      if (!(sd == 0 ? want0 : want1)) continue;
      const int ls = sd == 0 ? sl0 : sl1;
      const int fi = sd == 0 ? f0 : f1, bi = sd == 0 ? b0 : b1;
      bool ok = true;
      if (fi >= 0) {
        const R sf = (R)C.s(fi);
        const R lf = (R)T.P[m_prof(C.meta(fi))].len;
        const R gf = M::sub(M::sub(sf, s), lf);
        if (GUARD && fabsf((float)gf) <= kEpsPos * (float)(fabs(sf - s) + lf)) g.hit = true;
        if (!(gf >= (R)0)) ok = false;                   // L17 (2)
      }
      if (ok && bi >= 0) {
        const R sb = (R)C.s(bi);
        const R gb = M::sub(M::sub(s, sb), p.len);
        const R gbs = fabs(s - sb) + p.len;
        if (GUARD && fabsf((float)gb) <= kEpsPos * (float)gbs) g.hit = true;
        if (!(gb >= (R)0)) ok = false;                   // L17 (2)
        if (ok) {
          const PV<R> pb = pvals(T.P[m_prof(C.meta(bi))], (R)0);
          const R vb = (R)C.v(bi);
          const R v0b = (pb.vmax < (R)T.vmax[ls]) ? pb.vmax : (R)T.vmax[ls];
          const R an = idm<R, GUARD>(vb, v0b, true, gb, M::sub(vb, v), pb, b_hard, gbs, g);
          if (GUARD && fabsf((float)(an + (R)A.b_safe)) <= kEpsAcc) g.hit = true;
          if (!(an >= -(R)A.b_safe)) ok = false;         // L17 (1)
          if (sd == 0) anew0 = an; else anew1 = an;
        }
      } else if (ok) {
        const R mrg = M::sub(s, p.len);
        if (GUARD && fabsf((float)mrg - (float)A.start_margin) <= kEpsPos * ((float)s + (float)A.start_margin))
          g.hit = true;
        if (!(mrg >= (R)A.start_margin)) ok = false;    // L17 (3) lane-start rule
      }
      if (sd == 0) adm0 = ok; else adm1 = ok;
    }
    if (inG && (adm0 || adm1)) {                         // discretionary: utilities + draw
      R a_of = (R)0, a_of_new = (R)0;                    // old follower (L10)
      if (of >= 0) {
        const PV<R> po = pvals(T.P[m_prof(C.meta(of))], (R)0);
        const R so = (R)C.s(of), vo = (R)C.v(of);
        const R v0o = (po.vmax < (R)T.vmax[l]) ? po.vmax : (R)T.vmax[l];
        a_of = idm<R, GUARD>(vo, v0o, true, M::sub(M::sub(s, so), p.len), M::sub(vo, v), po,
                             b_hard, fabs(s - so) + p.len, g);
        const int li = lead >= 0 ? lead : i;             // free road if the ego has no leader
        const R sl_ = (R)C.s(li);
        const R ll_ = (R)T.P[m_prof(C.meta(li))].len;
        a_of_new = idm<R, GUARD>(vo, v0o, lead >= 0, M::sub(M::sub(sl_, so), ll_),
                                 M::sub(vo, (R)C.v(li)), po, b_hard, fabs(sl_ - so) + ll_, g);
      }
#pragma unroll 1
      for (int sd = 0; sd < 2; ++sd) {
        if (!(sd == 0 ? adm0 : adm1)) continue;
        const int ls = sd == 0 ? sl0 : sl1;
        const int fi = sd == 0 ? f0 : f1, bi = sd == 0 ? b0 : b1;
        R a_nf = (R)0;
        if (bi >= 0) {                                   // new follower before the change
          const PV<R> pb = pvals(T.P[m_prof(C.meta(bi))], (R)0);
          const R sb = (R)C.s(bi), vb = (R)C.v(bi);
          const R v0b = (pb.vmax < (R)T.vmax[ls]) ? pb.vmax : (R)T.vmax[ls];
          const int fj = fi >= 0 ? fi : bi;              // free road if no front
          const R sf = (R)C.s(fj);
          const R lf = (R)T.P[m_prof(C.meta(fj))].len;
          a_nf = idm<R, GUARD>(vb, v0b, fi >= 0, M::sub(M::sub(sf, sb), lf),
                               M::sub(vb, (R)C.v(fj)), pb, b_hard, fabs(sf - sb) + lf, g);
        }
        const R pol = M::add(M::sub(sd == 0 ? anew0 : anew1, a_nf), M::sub(a_of_new, a_of));
        if (sd == 0) pol0 = pol; else pol1 = pol;
      }
      {
        // U53 of Philox4x32-10(seed; vid, t) (ledger L16)
        const uint64_t sd = A.veh_seed ? A.veh_seed[me.vid] : A.seed;
        uint32_t c0 = A.rng_id ? (uint32_t)A.rng_id[me.vid] : (uint32_t)me.vid;
        uint32_t c1 = (uint32_t)T.t, c2 = 0u, c3 = 0u;
        uint32_t k0 = (uint32_t)(sd & 0xffffffffull), k1 = (uint32_t)(sd >> 32);
#pragma unroll
        for (int rr = 0; rr < 10; ++rr) {
          uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
          uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
          uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
          c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
          k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
        }
        const uint64_t mant = ((uint64_t)(c0 >> 5) << 26) + (uint64_t)(c1 >> 6);
        r = (double)mant * (1.0 / 9007199254740992.0);
      }
    }
  }
  SideRes<R> sr;
  sr.choice = -1;
  sr.hit = false;
  if (adm0 || adm1)                                      // O7 decision
    sr = lane_change<R, GUARD>(A, T, C, adm0, adm1, inG, mand, sl0, sl1, f0, f1, s, v, p, me,
                               a_cur, pol0, pol1, r);
  if (sr.hit) g.hit = true;
  return sr;
}

// O8-O9 for one vehicle given its acceleration and clamp (after O7): the
// ballistic update, the clamp, hand-off and arrival, the wait counter.
template <typename R, bool GUARD>
__device__ __forceinline__ void integrate(const StepArgs &A, const TileSh &T, R s, R v,
                                          const Me &me, const LEv<R> &use, int lc, int new_l,
                                          int wait0, Res &o, Guard &g) {
  using M = Ar<R>;
  o.nxt = me.nxt;
  o.nxt2 = me.nxt2;
  // O8 integrate (ledger L1) + clamp (L22, L23).  The fp64 path follows the
  // canonical sequence (position s1); the fp32 path carries the position as
  // base + advance so that stop-line / hand-off decisions and the residual
  // after a hand-off are free of cancellation at large s.
  const R a = use.a;
  const R vr = M::add(v, a);
  R s1, v1, adv;
  const bool adv_zero = (v == (R)0) && (vr <= (R)0);     // exact in both precisions
  if (vr < (R)0) {
    const R q = M::div(M::mul(v, v), M::mul((R)2, a));
    s1 = M::sub(s, q);
    adv = -q;
    v1 = (R)0;
  } else {
    adv = M::mul(M::add(v, vr), (R)0.5);
    s1 = M::add(s, adv);
    v1 = vr;
  }
  if (use.has_lim) {
    bool bind;
    if (M::fp64) {
      bind = s1 > use.lim;
    } else {
      bind = adv > use.limrel;
      if (GUARD && !adv_zero && fabsf((float)(adv - use.limrel)) <= kEpsPos * (float)(fabs(adv) + fabs(use.limrel) + (R)1e-3))
        g.hit = true;
    }
    if (bind) {
      if (GUARD && fabsf((float)use.limrel) <= kEpsPos * (float)(fabs(s) + fabs(use.lim)))
        g.hit = true;
      if (M::fp64 ? (use.lim < s) : (use.limrel < (R)0)) { s1 = s; adv = (R)0; v1 = (R)0; }
      else { s1 = use.lim; adv = use.limrel; v1 = (use.vlim < v1) ? use.vlim : v1; }
    }
  }
  // O9 hand-off and arrival (ledger L26, L31); position = pb + pa.
  // The lanes a vehicle reaches in the common case are resolved from the
  // tile's own tables: its road lane -> a junction lane of the tile (the
  // next1 hint) -> that junction lane's exit lane (length, inbox, staged by
  // k_prep); only a vehicle crossing further reads the global graph.  The
  // next lane after the exit lane is looked up only when it can matter (the
  // vehicle reaches the exit lane's end, or is within the guard band of it).
  R pb = M::fp64 ? s1 : s;
  R pa = M::fp64 ? (R)0 : adv;
  int curg = T.glob[new_l], ri = me.cur, n = use.next1, hand = 0;
  int cl = new_l, cx = -1;                              // current lane: local index / via exit of cx
  int nl = use.nl1;                                     // n as a local junction lane (-1 unknown)
  bool croad = T.isroad[new_l];
  R Lc = (R)T.len[new_l];
  bool fin = false;
  constexpr int kUnknown = -100;
  for (;;) {
    const bool dest_road = croad && route_at(A, me.vid, me.cur, me.nxt, me.nxt2, ri + 1) < 0;
    if (dest_road) {
      const R es = (R)me.ends;
      const R rem = M::sub(es, pb);
      if (GUARD && !(adv_zero && hand == 0) &&
          fabsf((float)(pa - rem)) <= kEpsPos * (float)(fabs(pa) + fabs(rem) + (R)1e-3))
        g.hit = true;
      if (pa >= rem) { fin = true; break; }
    }
    const R rem = M::sub(Lc, pb);
    const bool close = GUARD && !(adv_zero && hand == 0) &&
                       fabsf((float)(pa - rem)) <= kEpsPos * (float)(fabs(pa) + fabs(rem) + (R)1e-3);
    if (n == kUnknown && (pa > rem || close)) {           // next lane of a road lane beyond the tile
      const int R1 = route_at(A, me.vid, me.cur, me.nxt, me.nxt2, ri + 1);
      const int R2 = route_at(A, me.vid, me.cur, me.nxt, me.nxt2, ri + 2);
      n = next_from_road_any(A, T, curg, R1, R2);
      nl = -1;
    }
    if (close && n >= 0) g.hit = true;
    if (pa > rem && n >= 0) {
      pb = M::sub(pb, Lc);
      hand += 1;
      if (cl >= 0 && croad && nl >= 0) {                  // own road lane -> own junction lane
        curg = n;
        cl = nl;
        cx = -1;
        croad = false;
        Lc = (R)T.len[nl];
        n = xl_of(T, nl);
        nl = -1;
      } else if (cl >= 0 && !croad) {                    // own junction lane -> its exit lane
        const ExtFirst &x = T.ext[cl - T.nroad];
        curg = n;
        cx = cl;
        cl = x.dtile == T.tile ? x.dlocal : -1;
        croad = true;
        Lc = (R)x.Lb;
        ri += 1;
        n = kUnknown;
      } else {                                            // elsewhere: the global graph
        curg = n;
        cx = -1;
        cl = __ldg(A.lane_tile + curg) == T.tile ? (int)A.lane_local[curg] : -1;
        croad = __ldg(A.lane_road + curg) >= 0;
        Lc = (R)__ldg(A.lane_len + curg);
        if (croad) {
          ri += 1;
          n = kUnknown;
        } else {
          n = __ldg(A.exit_lane + curg);
        }
        nl = -1;
      }
      if (cl >= 0 && croad && n == kUnknown) {            // back on a road lane of this tile
        const int R1 = route_at(A, me.vid, me.cur, me.nxt, me.nxt2, ri + 1);
        const int R2 = route_at(A, me.vid, me.cur, me.nxt, me.nxt2, ri + 2);
        const Next nx = R1 < 0 ? Next{kLaneDest, false, -1} : next1_t(A, T, cl, R1, R2);
        n = nx.j;
        nl = nx.hint;
      }
      continue;
    }
    break;
  }
  s1 = M::fp64 ? pb : (hand == 0 ? s1 : M::add(pb, pa));
  const R vw = (R)A.v_wait;
  if (GUARD && fabsf((float)(v1 - vw)) <= kEpsV * (float)(fabs(v) + fabs(a) + (R)1)) g.hit = true;
  o.wait1 = wait0 + ((v1 < vw) ? 1 : 0);                 // ledger L28
  o.s1 = (float)s1;
  o.v1 = (float)v1;
  o.acc = (float)a;
  o.lane_g = curg;
  o.cursor = ri;
  o.cl = cl;
  o.cx = cx;
  o.lc = lc;
  o.hand = hand;
  o.fin = fin;
}

template <typename R, bool GUARD>
__device__ void veh_update(const StepArgs &A, const TileSh &T, const View &C, int i, Res &o,
                           Guard &g) {
  const uint32_t meta = C.meta(i);
  const int l = m_lane(meta), pr = m_prof(meta);
  Me me;
  me.vid = C.vid(i);
  me.cur = m_cursor(meta);
  me.nxt = C.nxt(i);                                     // ego-only fields
  me.nxt2 = C.nxt2(i);
  me.ends = C.ends(i);
  const int wait0 = C.wait(i);
  const PV<R> p = pvals(T.P[pr], (R)0);
  const R s = (R)C.s(i), v = (R)C.v(i);
  const int lead = (i + 1 < T.seg_end[l]) ? i + 1 : -1;
  // recorded decisions (test mode) go straight to their arrays
  if (A.record) {
    const int of = (i > T.seg_start[l]) ? i - 1 : -1;
    A.r_of[me.vid] = of >= 0 ? C.vid(of) : -1;
    for (int q = 0; q < 4; ++q) A.r_side[4 * me.vid + q] = -1;
  }
  Elig E;
  E.sl0 = E.sl1 = -1;
  E.mand = 0;
  E.inG = true;
  E.want0 = E.want1 = false;
  me.k = -1;
  if (T.isroad[l]) E = lc_elig<R, GUARD>(A, T, l, s, v, p, me, g);   // no LC in junction lanes
  LEv<R> use = eval_lane<R, GUARD>(A, T, C, l, lead, s, v, p, me, g);   // O4-O6
  if (A.record) {
    A.r_leader[me.vid] = use.leader;
    A.r_hops[me.vid] = (int8_t)use.hops;
    A.r_phantom[me.vid] = (int8_t)use.phantom;
  }
  int lc = 0, new_l = l;
  if (E.want0 || E.want1 || (A.record && T.isroad[l])) {
    const SideRes<R> sr = lc_decide<R, GUARD>(A, T, C, i, l, s, v, p, me, E, use.a, g);
    if (sr.choice >= 0) {
      use.a = sr.a;
      use.has_lim = sr.has_lim;
      use.lim = sr.lim;
      use.limrel = sr.limrel;
      use.vlim = sr.vlim;
      use.next1 = sr.next1;
      use.nl1 = sr.nl1;
      lc = sr.choice == 0 ? -1 : 1;
      new_l = sr.choice == 0 ? E.sl0 : E.sl1;
    }
  }
  integrate<R, GUARD>(A, T, s, v, me, use, lc, new_l, wait0, o, g);
}

}  // namespace sim
