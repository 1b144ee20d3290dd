// kernels.cu — the fused step kernel (a0-a4, a6) and the signal kernel (a5).
//
// k_step: one CTA per road tile.  Per step and tile:
//   1. merge the in-order stayers (slab) with the sorted inbox into the tile
//      snapshot in shared memory (a1; the paper's index update K3, P:130,
//      without a global sort: stayers cannot overtake, movers are few);
//   2. every thread updates one vehicle (a2 lookup, a3 IDM + MOBIL + signal,
//      a4 integrate / hand-off / arrival) reading only the snapshot;
//   3. stayers are compacted in order into the output slab (coalesced),
//      movers are appended to the destination tile's inbox, arrivals retired;
//   4. per-lane first-vehicle summaries for step t+1 are built with 64-bit
//      integer atomicMin (order independent), departures are inserted (K11,
//      P:142), and per-tile int64 counters accumulate (a6).
#include <cuda_runtime.h>

#include <algorithm>

#include "dev.h"
#include "model.cuh"

namespace sim {

__device__ __forceinline__ unsigned long long vkey(float s, int vid) {
  return ((unsigned long long)__float_as_uint(s) << 32) | (unsigned)vid;
}
// composite order key (lane_local, s, vid)
__device__ __forceinline__ unsigned long long hikey(int lane, float s) {
  return ((unsigned long long)(unsigned)lane << 32) | __float_as_uint(s);
}
__device__ __forceinline__ bool key_less(unsigned long long h1, int v1, unsigned long long h2,
                                         int v2) {
  return h1 < h2 || (h1 == h2 && v1 < v2);
}

// fp64 canonical path (exact_mode and guard fallback) kept out of line so the
// hot fp32 path is register-allocated on its own
__device__ __forceinline__ void record(const StepArgs &A, int vid, const Res &r, bool guard) {
  A.r_lc[vid] = (int8_t)r.lc;
  A.r_hand[vid] = (int8_t)(r.hand > 127 ? 127 : r.hand);
  A.r_acc[vid] = r.acc;
  A.r_fin[vid] = (int8_t)r.fin;
  A.r_guard[vid] = (uint8_t)(guard ? 1 : 0);
  A.r_mark[vid] = 1;
}

__device__ __forceinline__ void put_inbox(InboxRec *dst, const InboxRec &rec) {
  int4 *d = reinterpret_cast<int4 *>(dst);
  const int4 *s = reinterpret_cast<const int4 *>(&rec);
  d[0] = s[0];
  d[1] = s[1];
}

// Cold paths (inboxes larger than kSmemInbox, i.e. bulk lane changes after a
// setter or a load): kept out of line so they do not occupy the I-cache.
__device__ __noinline__ void rank_inbox_global(const InboxRec *inb, int n_in, int *bsort,
                                               int lane_id) {
  for (int j = lane_id; j < n_in; j += kThreads) {
    const InboxRec r = inb[j];
    const unsigned long long h = hikey(m_lane(r.meta), r.s);
    int rank = 0;
    for (int q = 0; q < n_in; ++q) {
      const InboxRec o = inb[q];
      rank += key_less(hikey(m_lane(o.meta), o.s), o.vid, h, r.vid);
    }
    bsort[rank] = j;
  }
}
__device__ __noinline__ int lower_bound_inbox_global(const InboxRec *inb, const int *bsort,
                                                     int n_in, unsigned long long h, int vid) {
  int lo = 0, hi = n_in;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const InboxRec o = inb[bsort[mid]];
    if (key_less(hikey(m_lane(o.meta), o.s), o.vid, h, vid)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// fire-and-forget 64-bit add (RED: no load round trip at the end of a tile)
__device__ __forceinline__ void red_add(long long *p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long *>(p), (unsigned long long)v);
}

struct Acc8 {                        // per-thread counters of one tile
  long long delay = 0;               // (travel / wait sums of arrivals go straight to tacc)
  int fin = 0, lc = 0, hand = 0, guard = 0, ovf = 0, ins = 0;
};

// Direct transport (NEXT-2): a mover entering another partition's
// tile is stored straight into the owner's inbox for t+1 and folded into the
// owner's summary / lane count with the same integer atomics a local mover
// uses, so no exchange or absorb step follows.  Returns 1 on inbox overflow.
__device__ __noinline__ int emit_peer(const StepArgs &A, const InboxRec &rec, int owner, int dt,
                                      int lane_g) {
  const PeerView &Q = A.peers[owner];
  const int nb = (A.t + 1) & 1, ns = (A.t + 1) % 3;
  const int vid = rec.vid;
  const int slot = atomicAdd(&Q.icnt[nb][dt], 1);
  int ovf = 0;
  if (slot < A.tile_icap[dt]) put_inbox(Q.inbox[nb] + A.tile_ibase[dt] + slot, rec);
  else ovf = 1;
  atomicMin(&Q.summ[ns][lane_g], vkey(rec.s, vid));
  Q.pubv[nb][vid] = rec.v;
  if (A.lane_cnt_next) atomicAdd(&Q.lcnt[ns][lane_g], 1);
  Q.insert_time[vid] = A.insert_time[vid];
  Q.status[vid] = ST_DRIVING;
  return ovf;
}

// a vehicle that leaves its slot: lane change / hand-off (kind 2, also every
// guard-deferred vehicle) or arrival (kind 3)
__device__ __forceinline__ void emit_moved(const StepArgs &A, const View &C, int i, const Res &r,
                                           int kind, Acc8 &acc, int tile) {
  const int vid = C.vid(i);
  acc.lc += r.lc != 0;
  acc.hand += r.hand;
  if (kind == 3) {
    A.status[vid] = ST_FINISHED;
    A.arrive_time[vid] = A.t + 1;
    A.wait_fin[vid] = r.wait1;
    acc.fin += 1;
    // int64 sums straight into the tile's accumulators (arrivals are rare; no
    // 64-bit register state through the update loop)
    long long *ta = A.tacc + (size_t)tile * kNAcc;
    atomicAdd(reinterpret_cast<unsigned long long *>(ta + ACC_SUM_TRAVEL),
              (unsigned long long)(long long)(A.t + 1 - A.insert_time[vid]));
    atomicAdd(reinterpret_cast<unsigned long long *>(ta + ACC_SUM_WAIT_FIN), (unsigned long long)(long long)r.wait1);
    return;
  }
  const uint32_t meta = C.meta(i);
  const int cur = m_cursor(meta);
  InboxRec rec;
  rec.s = r.s1;
  rec.v = r.v1;
  rec.vid = vid;
  rec.nxt = route_at(A, vid, cur, r.nxt, r.nxt2, r.cursor + 1);
  rec.nxt2 = route_at(A, vid, cur, r.nxt, r.nxt2, r.cursor + 2);
  rec.meta = pack_meta(A.lane_local[r.lane_g], m_prof(meta), r.cursor);
  rec.wait = r.wait1;
  rec.pad = 0;
  const int dt = A.lane_tile[r.lane_g];
  const int owner = A.tile_owner[dt];
  if (owner == A.rank) {
    const int slot = atomicAdd(&A.icnt_out[dt], 1);
    if (slot < A.tile_icap[dt]) put_inbox(A.inbox_out + A.tile_ibase[dt] + slot, rec);
    else acc.ovf += 1;
    atomicMin(&A.summ_next[r.lane_g], vkey(r.s1, vid));
    A.pubv_next[vid] = r.v1;
    if (A.lane_cnt_next) atomicAdd(&A.lane_cnt_next[r.lane_g], 1);
  } else if (A.peers) {                             // direct transport (NEXT-2)
    acc.ovf += emit_peer(A, rec, owner, dt, r.lane_g);
  } else {                                          // migrant to another partition
    const int slot = atomicAdd(&A.out_cnt[owner], 1);
    if (slot < A.out_cap[owner]) {
      MigRec *m = A.out_buf + A.out_off[owner] + 1 + slot;
      put_inbox(&m->rec, rec);
      m->tile = dt;
      m->insert_time = A.insert_time[vid];
    } else {
      acc.ovf += 1;
    }
  }
}

struct StepShared {
  TileSh T;
  unsigned long long bk_hi[kSmemInbox];       // inbox keys (arrival order)
  int bk_vid[kSmemInbox];
  int bsort[kSmemInbox];
  unsigned long long sk_hi[kSmemInbox];       // inbox keys in sorted order
  int sk_vid[kSmemInbox];
};

#ifndef KSTEP_WARPS
#define KSTEP_WARPS 1
#endif
#ifndef KSTEP_MINB
#define KSTEP_MINB (32 / KSTEP_WARPS)
#endif
constexpr int kStepWarps = KSTEP_WARPS;

// What the phases of one tile hand to each other (registers of its warp).
struct TileCtx {
  int tile, n, base, ibase, nl, nroad;
  View C;
};

// Phase 1 of a road tile (one warp; intra-tile synchronisation is __syncwarp()):
// tile metadata and the merged snapshot (a1).
template <bool EXACT>
__device__ __forceinline__ void tile_load(const StepArgs &A, StepShared &S, unsigned char *dyn,
                                          TileCtx &x, const int lane_id) {
  TileSh &T = S.T;
  // ---- tile metadata -----------------------------------------------------
  // One coalesced read of the tile descriptor (host-built): lane
  // ids / lengths / speed limits / usable flags and every road-lane successor
  // with its target road, exit lane and the exit lane's reachable roads.
  const int tile = x.tile;
  const int doff = A.desc_off[tile], dend = A.desc_off[tile + 1];
  const int n_st = A.cnt_in[tile];
  const int n_in = A.icnt_in[tile];
  const int n = n_st + n_in;
  const int base = A.tile_base[tile];
  const int ibase = A.tile_ibase[tile];
  // lane counts from the static tile tables (same load wave as the offsets),
  // so every descriptor word below is addressed without waiting for it
  const int nl = A.tile_lane_off[tile + 1] - A.tile_lane_off[tile], nroad = A.tile_nroad[tile];
  const int *W = A.desc + doff;                     // read straight from global (L2)
  int ew[8];                                        // successor entry of this lane (if any)
  {
    const int eo = 4 + 4 * nl + 6 * nroad + 8 * lane_id;
    if (doff + eo + 8 <= dend) {
#pragma unroll
      for (int q = 0; q < 8; ++q) ew[q] = W[eo + q];
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) ew[q] = 0;
    }
  }
  const int ne = W[2];
  // lane records, the per-road-lane group tables and the (host-sorted) usable
  // successors go straight into the tile's shared metadata; only the stop bit
  // (signal of the junction lane at t) is computed here
  if (lane_id == 0) {
    T.nl = nl;
    T.nroad = nroad;
    T.tile = tile;
    T.base = base;
    T.ibase = ibase;
    T.cap = A.tile_cap[tile];
    T.icap = A.tile_icap[tile];
  }
  if (lane_id < nl) {
    const int l = lane_id;
    const int fl = W[4 + 3 * nl + l];
    T.glob[l] = W[4 + l];
    T.len[l] = __int_as_float(W[4 + nl + l]);
    T.vmax[l] = __int_as_float(W[4 + 2 * nl + l]);
    T.isroad[l] = l < nroad;
    T.usable[l] = fl & 1;
    T.seg_start[l] = 0;
    T.seg_end[l] = 0;
    T.first_out[l] = 0x7fffffff;
    // road lanes are the first nroad local lanes, leftmost first (validated at create)
    T.left[l] = (l < nroad && l > 0) ? (int8_t)(l - 1) : (int8_t)-1;
    T.right[l] = (l < nroad - 1) ? (int8_t)(l + 1) : (int8_t)-1;
    if (l < nroad) {
      const int *gw = W + 4 + 4 * nl + 6 * l;
      T.sn[l] = (uint8_t)((fl >> 8) & 0xff);
      T.ng[l] = (uint8_t)((fl >> 16) & 0xff);
      const unsigned g4 = (unsigned)gw[0];
      T.gbeg[l][0] = (uint8_t)g4;
      T.gbeg[l][1] = (uint8_t)(g4 >> 8);
      T.gbeg[l][2] = (uint8_t)(g4 >> 16);
      T.gbeg[l][3] = (uint8_t)(g4 >> 24);
      T.gbeg[l][4] = (uint8_t)gw[1];
#pragma unroll
      for (int q = 0; q < kMaxGroups; ++q) T.gtroad[l][q] = gw[2 + q];
    }
  }
  if (lane_id < ne) {
    const int fl = ew[3];
    SuccEnt e;
    e.j = ew[0];
    e.troad = ew[1];
    e.b = ew[2];
    e.outr = make_int4(ew[4], ew[5], ew[6], ew[7]);
    e.stop = ((fl & 1) && A.lane_sig[e.j] != SIG_GREEN) ? 1 : 0;
    T.se[(fl >> 8) & 0xff][fl >> 16] = e;
  }
  reinterpret_cast<int16_t *>(&T.gidx[0][0])[lane_id] = (int16_t)-1;    // 64 bytes
  __syncwarp();
  {
    // distinct target roads of the road lanes (entry e = lane a, group g),
    // numbered in order of first appearance; per road a lane bitmask
    static_assert(kMaxRoadLanes * kMaxGroups <= 32, "one entry per thread");
    const int a = lane_id / kMaxGroups, g = lane_id % kMaxGroups;
    const bool valid = a < nroad && g < T.ng[a];
    const int R = valid ? T.gtroad[a][g] : -1;
    const unsigned vb = __ballot_sync(0xffffffffu, valid);
    bool first = valid;
    int myk = -1;
    unsigned fb = 0;
#pragma unroll 1
    for (int q = 0; q < kMaxRoadLanes * kMaxGroups; ++q) {
      const int Rq = __shfl_sync(0xffffffffu, R, q);
      if (valid && ((vb >> q) & 1u) && Rq == R && q < lane_id) first = false;
    }
    fb = __ballot_sync(0xffffffffu, first);
#pragma unroll 1
    for (int q = 0; q < kMaxRoadLanes * kMaxGroups; ++q) {
      const int Rq = __shfl_sync(0xffffffffu, R, q);
      if (valid && ((fb >> q) & 1u) && Rq == R) myk = __popc(fb & ((1u << q) - 1u));
    }
    if (first) T.troad[myk] = R;
    if (valid) T.gidx[a][myk] = (int8_t)g;
    const int ntr = __popc(fb);
    for (int k = 0; k < ntr; ++k) {
      const unsigned m = __ballot_sync(0xffffffffu, valid && myk == k);
      unsigned lanes = 0;
#pragma unroll
      for (int aa = 0; aa < kMaxRoadLanes; ++aa)
        if ((m >> (aa * kMaxGroups)) & ((1u << kMaxGroups) - 1u)) lanes |= 1u << aa;
      if (lane_id == 0) T.reach[k] = (uint8_t)lanes;
    }
    const unsigned um = __ballot_sync(0xffffffffu, lane_id < nroad && T.usable[lane_id]);
    if (lane_id == 0) { T.ntr = ntr; T.umask = um; }
  }
  __syncwarp();

  // snapshot view: shared memory, or this tile's global scratch if too large
  View C;
  const bool smem_ok = (n <= kSmemVeh) && (n_in <= kSmemInbox);
  if (smem_ok) {
    C.p = reinterpret_cast<uint32_t *>(dyn);
    C.sp = reinterpret_cast<int16_t *>(dyn + kSmemVeh * 16);
    C.st = kSmemVeh;
  } else {                                   // scratch region of the tile: 5 x (cap + icap) words
    C.st = T.cap + T.icap;
    C.p = A.scratch + 5 * (size_t)(base + ibase);
    C.sp = reinterpret_cast<int16_t *>(C.p + 4 * C.st);
  }
  int *bsort = (n_in <= kSmemInbox) ? S.bsort : (A.bsort_scratch + ibase);
  const InboxRec *inb = A.inbox_in + ibase;
  const bool small_in = n_in <= kSmemInbox;

  // ---- 1. merge stayers + sorted inbox (a1) ---------------------------------
  if (n_in > 0) {
    if (small_in) {
      for (int j = lane_id; j < n_in; j += kThreads) {
        const InboxRec r = inb[j];
        S.bk_hi[j] = hikey(m_lane(r.meta), r.s);
        S.bk_vid[j] = r.vid;
      }
      __syncwarp();
      for (int j = lane_id; j < n_in; j += kThreads) {
        const unsigned long long h = S.bk_hi[j];
        const int vj = S.bk_vid[j];
        int rank = 0;
        for (int q = 0; q < n_in; ++q) rank += key_less(S.bk_hi[q], S.bk_vid[q], h, vj);
        bsort[rank] = j;
        S.sk_hi[rank] = h;
        S.sk_vid[rank] = vj;
      }
    } else {
      rank_inbox_global(inb, n_in, bsort, lane_id);
    }
  }
  __syncwarp();
  // stayers: position = own index + #inbox keys below (binary search in the sorted inbox).
  // Two slab rows per iteration, loads issued before the stores (more bytes in flight).
  for (int i0 = lane_id; i0 < n_st; i0 += 2 * kThreads) {
    float sv[2], vv[2];
    uint32_t mv[2];
    int idv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * kThreads;
      if (i < n_st) {
        const int gi = base + i;
        sv[u] = A.in.s[gi]; vv[u] = A.in.v[gi]; mv[u] = A.in.meta[gi]; idv[u] = A.in.vid[gi];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
    const int i = i0 + u * kThreads;
    if (i >= n_st) break;
    const float s = sv[u];
    const uint32_t meta = mv[u];
    const int vid = idv[u];
    int pos = i;
    if (n_in > 0) {
      const unsigned long long h = hikey(m_lane(meta), s);
      int lo = 0, hi = n_in;
      if (small_in) {
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (key_less(S.sk_hi[mid], S.sk_vid[mid], h, vid)) lo = mid + 1; else hi = mid;
        }
      } else {
        lo = lower_bound_inbox_global(inb, bsort, n_in, h, vid);
      }
      pos += lo;
    }
    C.s(pos) = s;
    C.v(pos) = vv[u];
    C.vid(pos) = vid;
    C.meta(pos) = meta;
    C.src(pos) = (int16_t)i;
    }
  }
  // inbox records: position = sorted rank + #stayers below (binary search in the slab)
  for (int r = lane_id; r < n_in; r += kThreads) {
    const int j = bsort[r];
    const InboxRec rec = inb[j];
    const unsigned long long h = hikey(m_lane(rec.meta), rec.s);
    int lo = 0, hi = n_st;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int gi = base + mid;
      if (key_less(hikey(m_lane(A.in.meta[gi]), A.in.s[gi]), A.in.vid[gi], h, rec.vid)) lo = mid + 1;
      else hi = mid;
    }
    const int pos = r + lo;
    C.s(pos) = rec.s;
    C.v(pos) = rec.v;
    C.vid(pos) = rec.vid;
    C.meta(pos) = rec.meta;
    C.src(pos) = (int16_t)(-j - 1);
  }
  __syncwarp();
  // lane segments of the snapshot
  for (int i = lane_id; i < n; i += kThreads) {
    const int l = m_lane(C.meta(i));
    if (i == 0 || m_lane(C.meta(i - 1)) != l) T.seg_start[l] = i;
    if (i == n - 1 || m_lane(C.meta(i + 1)) != l) T.seg_end[l] = i + 1;
  }
  __syncwarp();
  x.n = n;
  x.base = base;
  x.ibase = ibase;
  x.nl = nl;
  x.nroad = nroad;
  x.C = C;
}

  // ---- 2-3. per-vehicle update (a2-a4) and outputs, 32 vehicles at a time ----
  // fp32 path: vehicles whose decision margins fall inside the guard band are
  // deferred and recomputed after the loop with the canonical fp64 sequence;
  // they leave through the inbox (as movers), so the in-order compaction of the
  // stayers never waits for them and the fp64 code stays out of the hot loop.
template <bool EXACT>
__device__ __forceinline__ void tile_update(const StepArgs &A, StepShared &S, const TileCtx &x,
                                            Acc8 &acc, int &run, int &ndef, const int lane_id) {
  TileSh &T = S.T;
  const int n = x.n, base = x.base, ibase = x.ibase;
  const View C = x.C;
  int *dlist = A.dl_scratch + base + ibase;
  for (int c0 = 0; c0 < n; c0 += kThreads) {
    const int i = c0 + lane_id;
    Res r;
    int kind = 0;                                   // 0 none, 1 stayer, 2 mover, 3 finished
    bool defer = false;
    if (i < n) {
      if constexpr (EXACT) {
        Guard g;
        g.hit = false;
        g.why = 0;
        veh_update<double, false>(A, T, C, i, r, g);
      } else {
        Guard g;
        g.hit = false;
        g.why = 0;
        veh_update<float, true>(A, T, C, i, r, g);
        defer = g.hit;
#ifdef GUARD_STATS
        if (g.hit)
          for (int b = 0; b < 32; ++b)
            if (g.why & (1u << b)) atomicAdd(&g_guard_stats[b], 1ull);
#endif
      }
      if (!defer) {
        if (A.record) record(A, C.vid(i), r, false);
        const int l = m_lane(C.meta(i));
        if (r.fin) kind = 3;
        else if (r.lc == 0 && r.hand == 0 && r.lane_g == T.glob[l]) kind = 1;
        else kind = 2;
      }
    }
    if constexpr (!EXACT) {
      const unsigned dball = __ballot_sync(0xffffffffu, defer);
      if (defer) dlist[ndef + __popc(dball & ((1u << lane_id) - 1u))] = i;
      ndef += __popc(dball);
    }
    // order-preserving compaction of stayers (warp ballot)
    const unsigned ball = __ballot_sync(0xffffffffu, kind == 1);
    if (kind == 1) {
      const int pos = base + run + __popc(ball & ((1u << lane_id) - 1u));
      const uint32_t meta = C.meta(i);
      A.out.s[pos] = r.s1;
      A.out.v[pos] = r.v1;
      A.out.vid[pos] = C.vid(i);
      A.out.nxt[pos] = r.nxt;
      A.out.nxt2[pos] = r.nxt2;
      A.out.meta[pos] = meta;
      A.out.wait[pos] = r.wait1;
      atomicMin(&T.first_out[m_lane(meta)], pos);
    } else if (kind >= 2) {
      emit_moved(A, C, i, r, kind, acc, x.tile);
    }
    run += __popc(ball);
  }
}

// The guard fallback of one deferred vehicle (fp64 canonical sequence, DESIGN
// §3.3), out of line: a real call keeps the fp64 code and its registers out
// of k_step<false>'s hot loop (C4: 277 -> 274 us).  Removing the fp64 path
// from k_step entirely measured 262 us, but a separate k_defer kernel that
// rebuilds the deferred tiles cost more (~28 us of single-warp latency).
__device__ __noinline__ void defer_recompute(const StepArgs &A, const TileSh &T, const View &C,
                                             int i, Acc8 &acc, int tile) {
  Res r;
  Guard g;
  g.hit = false;
  g.why = 0;
  veh_update<double, false>(A, T, C, i, r, g);
  if (A.record) record(A, C.vid(i), r, true);
  emit_moved(A, C, i, r, r.fin ? 3 : 2, acc, tile);
  acc.guard += 1;
}

// Phase 3: guard-deferred vehicles (fp64), lane summaries for t+1, departures
// and counters (a4, a6).
template <bool EXACT>
__device__ __forceinline__ void tile_finish(const StepArgs &A, StepShared &S, const TileCtx &x,
                                            Acc8 &acc, const int run, const int ndef,
                                            const int lane_id) {
  TileSh &T = S.T;
  const int tile = x.tile, n = x.n, base = x.base, ibase = x.ibase, nl = x.nl, nroad = x.nroad;
  const View C = x.C;
  int *dlist = A.dl_scratch + base + ibase;
  if constexpr (!EXACT) {
    __syncwarp();
    for (int q = lane_id; q < ndef; q += kThreads) defer_recompute(A, T, C, dlist[q], acc, tile);
  }
  __syncwarp();

  // ---- 4. summaries, insertions, counters ------------------------------------
  for (int l = lane_id; l < nl; l += kThreads) {
    const int g = T.glob[l];
    const int pos = T.first_out[l];
    if (pos != 0x7fffffff) {
      const float s1 = A.out.s[pos];
      const int vid = A.out.vid[pos];
      atomicMin(&A.summ_next[g], vkey(s1, vid));
      A.pubv_next[vid] = A.out.v[pos];
    }
    A.summ_clear[g] = kEmptyKey;
    if (A.lane_cnt_next && pos != 0x7fffffff) {     // stayers of lane l: [pos, next lane's first)
      int end = base + run;
      for (int q = l + 1; q < nl; ++q)
        if (T.first_out[q] != 0x7fffffff) { end = T.first_out[q]; break; }
      atomicAdd(&A.lane_cnt_next[g], end - pos);
    }
  }
  for (int l = lane_id; l < nroad; l += kThreads) { // departures (K11; ledger L25)
    const int g = T.glob[l];
    const int h = A.pend_head[g];
    if (h >= A.pend_off[g + 1]) continue;
    const int k = A.pend_vid[h];
    if (A.depart[k] > A.t || !T.usable[l]) continue;
    const double ss = (double)A.start_s[k];
    const Prof &pk = T.P[A.veh_prof[k]];
    const int a0 = T.seg_start[l], b0 = T.seg_end[l];
    const int fa = upper_bound_s(C, a0, b0, (float)ss);
    bool ok = true;
    if (fa < b0) {
      const double sa = C.s(fa), la = T.P[m_prof(C.meta(fa))].len_d;
      if (!(__dadd_rn(__dadd_rn(sa, -ss), -la) >= pk.s0_d)) ok = false;
    }
    if (fa > a0) {
      const int b = fa - 1;
      const Prof &pb = T.P[m_prof(C.meta(b))];
      const double need = __dadd_rn(__dadd_rn((double)C.v(b), __dmul_rn(0.5, pb.a_max_d)), pk.s0_d);
      if (!(__dadd_rn(__dadd_rn(ss, -(double)C.s(b)), -pk.len_d) >= need)) ok = false;
    } else {
      if (!(__dadd_rn(ss, -pk.len_d) >= A.start_margin)) ok = false;
    }
    if (!ok) continue;
    InboxRec rec;
    rec.s = (float)ss;
    rec.v = 0.f;
    rec.vid = k;
    const int off = A.route_start[k], rl = A.route_len[k];
    rec.nxt = rl > 1 ? A.route[off + 1] : -1;
    rec.nxt2 = rl > 2 ? A.route[off + 2] : -1;
    rec.meta = pack_meta(l, A.veh_prof[k], 0);
    rec.wait = 0;
    rec.pad = 0;
    const int slot = atomicAdd(&A.icnt_out[tile], 1);
    if (slot < T.icap) put_inbox(A.inbox_out + ibase + slot, rec);
    else acc.ovf += 1;
    atomicMin(&A.summ_next[g], vkey(rec.s, k));
    A.pubv_next[k] = 0.f;
    if (A.lane_cnt_next) atomicAdd(&A.lane_cnt_next[g], 1);
    A.pend_head[g] = h + 1;
    A.status[k] = ST_DRIVING;
    A.insert_time[k] = A.t + 1;
    if (A.record) A.r_ins[k] = 1;
    acc.ins += 1;
    acc.delay += (long long)(A.t + 1 - A.depart[k]);
  }
  // warp reduction of the counters (exact, order independent): 32-bit counts
  // with redux.sync; the int64 sums only in warps that saw an arrival / insertion
  const unsigned c_fin = __reduce_add_sync(0xffffffffu, (unsigned)acc.fin);
  const unsigned c_ins = __reduce_add_sync(0xffffffffu, (unsigned)acc.ins);
  const unsigned c_lc = __reduce_add_sync(0xffffffffu, (unsigned)acc.lc);
  const unsigned c_hand = __reduce_add_sync(0xffffffffu, (unsigned)acc.hand);
  const unsigned c_guard = __reduce_add_sync(0xffffffffu, (unsigned)acc.guard);
  const unsigned c_ovf = __reduce_add_sync(0xffffffffu, (unsigned)acc.ovf);
  long long s_delay = acc.delay;
  if (c_ins) {
    for (int o = 16; o > 0; o >>= 1) s_delay += __shfl_down_sync(0xffffffffu, s_delay, o);
  }
  if (lane_id == 0) {
    long long *ta = A.tacc + (size_t)tile * kNAcc;
    red_add(ta + ACC_VEH_STEPS, n);
    if (c_fin) red_add(ta + ACC_FINISHED, c_fin);
    if (c_ins) {
      red_add(ta + ACC_INSERTED, c_ins);
      red_add(ta + ACC_SUM_DELAY, s_delay);
    }
    if (c_lc) red_add(ta + ACC_LANE_CHANGES, c_lc);
    if (c_hand) red_add(ta + ACC_HANDOFFS, c_hand);
    if (c_guard) red_add(ta + ACC_GUARD, c_guard);
    if (c_ovf) red_add(ta + ACC_OVERFLOW, c_ovf);
    A.cnt_out[tile] = run;
    A.icnt_in[tile] = 0;
  }
}

// Persistent kernel.  A block of kStepWarps warps takes kStepWarps consecutive
// road tiles from a work counter (largest tiles first: A.tiles is sorted by slot
// capacity at create), one tile per warp, and runs the three phases of its
// tiles in step with block barriers in between, so all warps of an SM execute
// the same code at a time (the whole kernel does not fit the instruction
// cache) and issue their HBM loads together.  Consecutive tiles of the sorted
// list have similar sizes, so little time is lost at the barriers.  The last
// block to finish resets the counters for the next launch.
template <bool EXACT>
__global__ void __launch_bounds__(kStepWarps * kThreads, KSTEP_MINB)
    k_step(const __grid_constant__ StepArgs A) {
  extern __shared__ __align__(16) unsigned char dyn_all[];
  __shared__ StepShared SS[kStepWarps];
  __shared__ Prof prof[kSmemProf];
  __shared__ int s_base;
  const int warp = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
  StepShared &S = SS[warp];
  unsigned char *dyn = dyn_all + (size_t)warp * (kSmemVeh * 18);
  if (A.n_prof <= kSmemProf) {                      // profiles as int4 words (Prof is 96 B)
    const int nw = A.n_prof * (int)(sizeof(Prof) / 16);
    for (int q = threadIdx.x; q < nw; q += blockDim.x)
      reinterpret_cast<int4 *>(prof)[q] = reinterpret_cast<const int4 *>(A.prof)[q];
  }
  if (lane_id == 0) S.T.P = A.n_prof <= kSmemProf ? prof : A.prof;
  for (;;) {
    if (threadIdx.x == 0) s_base = atomicAdd(&A.work[0], kStepWarps);
    __syncthreads();
    const int b0 = s_base;
    if (b0 >= A.n_own) break;
    const int idx = b0 + warp;
    const bool has = idx < A.n_own;
    TileCtx x;
    x.tile = has ? A.tiles[idx] : 0;
    if (has) tile_load<EXACT>(A, S, dyn, x, lane_id);
    __syncthreads();
    Acc8 acc;
    int run = 0, ndef = 0;
    if (has) tile_update<EXACT>(A, S, x, acc, run, ndef, lane_id);
    __syncthreads();
    if (has) tile_finish<EXACT>(A, S, x, acc, run, ndef, lane_id);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&A.work[1], 1) == (int)gridDim.x - 1) {
      A.work[0] = 0;
      A.work[1] = 0;
    }
  }
}

// ---- a5: per-junction signal controller -------------
// One warp per junction.  Every lane runs the (tiny) phase machine on the same
// inputs; the MAX_PRESSURE choice is a warp reduction of the
// movement pressures count(pred) - count(succ) over the green slots of each
// phase; lane 0 stores the state, all lanes write the junction's signals.
__device__ __forceinline__ int sig_count(const SignalArgs &a, int lane) {
  if (!a.peers) return a.lane_cnt[lane];
  return a.peers[a.tile_owner[a.lane_tile[lane]]].lcnt[a.cnt_buf][lane];   // owner's count (NEXT-2)
}

__global__ void k_signal(SignalArgs a) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= a.n_junctions) return;
  const int K = a.ph_off[j + 1] - a.ph_off[j];
  const int j0 = a.jl_off[j], nj = a.jl_off[j + 1] - j0;
  int pol = a.policy[j], ph = a.phase[j];
  int el = a.elapsed[j], q = a.pending[j], y = a.yellow_left[j];
  const int preq = a.pol_request[j];
  if (preq >= 0 && K > 0 && preq != pol) {         // set_tl_policy first (L42)
    pol = preq;
    if (pol == POL_FIXED || pol == POL_MAXP) el = 0;
  }
  const int req = a.request[j];
  int rem = a.remaining[j];
  if (req >= 0) {                                   // requests apply before sig_t (L35)
    pol = POL_MANUAL;
    rem = -1;
    if (y > 0) q = req;
    else if (req != ph) {
      if (a.yellow > 0) { y = a.yellow; q = req; }
      else { ph = req; q = req; }
    }
  }
  const int dreq = a.dur_request[j];
  if (dreq >= 1 && K > 0) {                         // set_tl_duration (L43)
    pol = POL_MANUAL;
    rem = dreq;
  }
  // advance t -> t+1 (O11) into the stored state; sig_t uses (pol, ph, y) above
  int nph = ph, ny = y, nel = el, nq = q;
  if ((pol == POL_FIXED || pol == POL_MAXP) && K > 0) {
    if (ny > 0) {
      ny -= 1;
      if (ny == 0) { nph = nq; nel = 0; }
    } else {
      nel += 1;
      if (pol == POL_FIXED && nel >= a.green_steps[a.ph_off[j] + nph]) {
        const int nx = (nph + 1) % K;
        if (a.yellow > 0) { ny = a.yellow; nq = nx; }
        else { nph = nx; nq = nx; nel = 0; }
      } else if (pol == POL_MAXP && nel >= a.mp_period) {
        // movement pressures of this lane's slots, then per phase a warp sum
        const uint8_t *gr = a.green + a.green_off[j];
        int best = 0, best_p = 0;
        for (int k = 0; k < K; ++k) {
          int part = 0;
          for (int sl = lane; sl < nj; sl += 32)
            if (gr[(int64_t)k * nj + sl])
              part += sig_count(a, a.jl_pred[j0 + sl]) - sig_count(a, a.jl_succ[j0 + sl]);
          const int pk = __reduce_add_sync(0xffffffffu, part);
          if (k == 0 || pk > best_p) { best = k; best_p = pk; }     // ties -> lowest index
        }
        if (best == nph) nel = 0;                   // keep the green for another period
        else if (a.yellow > 0) { ny = a.yellow; nq = best; }
        else { nph = best; nq = best; nel = 0; }
      }
    }
  } else if (pol == POL_MANUAL) {
    if (ny > 0) {
      ny -= 1;
      if (ny == 0) nph = nq;
    } else if (rem > 0) {                           // hold d green steps, then the next phase
      rem -= 1;
      if (rem == 0) {
        const int nx = (nph + 1) % K;
        if (a.yellow > 0) { ny = a.yellow; nq = nx; }
        else { nph = nx; nq = nx; }
        rem = -1;
      }
    }
    nel += 1;
  }
  if (lane == 0) {
    if (req >= 0) a.request[j] = -1;
    if (preq >= 0) a.pol_request[j] = -1;
    if (dreq >= 0) a.dur_request[j] = -1;
    a.remaining[j] = rem;
    a.policy[j] = (uint8_t)pol;
    a.phase[j] = nph;
    a.elapsed[j] = nel;
    a.yellow_left[j] = ny;
    a.pending[j] = nq;
  }
  const uint8_t *grow = a.green + a.green_off[j] + (int64_t)ph * nj;
  for (int k = lane; k < nj; k += 32) {
    uint8_t sg;
    if (pol == POL_NONE || K == 0) sg = SIG_GREEN;
    else {
      const bool g = grow[k] != 0;
      sg = y > 0 ? (g ? SIG_YELLOW : SIG_RED) : (g ? SIG_GREEN : SIG_RED);
    }
    a.lane_sig[a.jl[j0 + k]] = sg;
  }
}

__global__ void k_apply_requests(int32_t *request, const int32_t *junc, const int32_t *phase, int m) {
  // entries are distinct junctions (the host keeps the last one per junction)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) request[junc[i]] = phase[i];
}

__global__ void k_reduce_acc(const long long *tacc, int n_tiles, const int32_t *cnt,
                             const int32_t *icnt, const uint8_t *status, int nv, long long *out) {
  // out (zeroed by the caller): [0, kNAcc) per-tile counters, kNAcc: driving
  // (stayers + inbox), kNAcc+1 / +2: PENDING / FINISHED vehicles from status
  __shared__ unsigned long long sh[kNAcc + 3];
  if (threadIdx.x < kNAcc + 3) sh[threadIdx.x] = 0;
  __syncthreads();
  const int stride = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  long long loc[kNAcc + 3] = {0};
  for (int t = t0; t < n_tiles; t += stride) {
#pragma unroll
    for (int c = 0; c < kNAcc; ++c) loc[c] += tacc[(size_t)t * kNAcc + c];
    loc[kNAcc] += cnt[t] + icnt[t];
  }
  for (int k = t0; k < nv; k += stride) {
    const uint8_t s = status[k];
    loc[kNAcc + 1] += s == ST_PENDING;
    loc[kNAcc + 2] += s == ST_FINISHED;
  }
#pragma unroll
  for (int c = 0; c < kNAcc + 3; ++c) {
    long long x = loc[c];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&sh[c], (unsigned long long)x);
  }
  __syncthreads();
  if (threadIdx.x < kNAcc + 3 && sh[threadIdx.x])
    atomicAdd(reinterpret_cast<unsigned long long *>(&out[threadIdx.x]), sh[threadIdx.x]);
}

// Per-group metrics (batched environments): the counters and driving counts
// of the own tiles, per group.  out [n_groups][kNAcc + 1] (zeroed by the caller).
__global__ void k_reduce_groups(const long long *tacc, const int32_t *tiles, int n_own,
                                const int32_t *tile_group, const int32_t *cnt,
                                const int32_t *icnt, long long *out) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_own; i += stride) {
    const int t = tiles[i];
    long long *o = out + (size_t)tile_group[t] * (kNAcc + 1);
    for (int c = 0; c < kNAcc; ++c) {
      const long long x = tacc[(size_t)t * kNAcc + c];
      if (x) atomicAdd(reinterpret_cast<unsigned long long *>(o + c), (unsigned long long)x);
    }
    const int d = cnt[t] + icnt[t];
    if (d) atomicAdd(reinterpret_cast<unsigned long long *>(o + kNAcc), (unsigned long long)d);
  }
}

__global__ void __launch_bounds__(128) k_lane_stats(StepArgs A, int32_t *cnt, int32_t *wt,
                                                   float *road_speed, float zone) {
  // lane queue length: per lane, vehicles and those with v < v_wait
  // within the last `zone` metres, over stayers + inbox of each own
  // tile; a lane belongs to one tile, so its totals are written, not added.
  // Road travelling speed: the tile's road lanes are its road.
  // One warp per tile (tiles hold ~100 vehicles), four tiles per block.
  __shared__ int sc_[4][kMaxTileLanes], sw_[4][kMaxTileLanes];
  __shared__ double sv_[4][kMaxTileLanes];
  __shared__ float slen_[4][kMaxTileLanes];          // lane lengths (read once per lane)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * 4 + w;
  if (idx >= A.n_own) return;
  int *sc = sc_[w], *sw = sw_[w];
  double *sv = sv_[w];
  float *slen = slen_[w];
  const int tile = A.tiles[idx];
  const int ns = A.cnt_in[tile], ni = A.icnt_in[tile];
  const int l0 = A.tile_lane_off[tile], nl = A.tile_lane_off[tile + 1] - l0;
  sc[lane] = sw[lane] = 0;
  sv[lane] = 0.0;
  if (lane < nl) slen[lane] = A.lane_len[A.tile_lanes[l0 + lane]];
  __syncwarp();
  const int base = A.tile_base[tile], ibase = A.tile_ibase[tile];
  for (int i = lane; i < ns + ni; i += 32) {
    float s, v;
    uint32_t meta;
    if (i < ns) {
      const int gi = base + i;
      s = A.in.s[gi]; v = A.in.v[gi]; meta = A.in.meta[gi];
    } else {
      const InboxRec r = A.inbox_in[ibase + i - ns];
      s = r.s; v = r.v; meta = r.meta;
    }
    const int l = m_lane(meta);
    atomicAdd(&sc[l], 1);
    if (road_speed) atomicAdd(&sv[l], (double)v);
    if (v < A.v_wait && (slen[l] - s) <= zone) atomicAdd(&sw[l], 1);
  }
  __syncwarp();
  if (lane < nl) {
    const int g = A.tile_lanes[l0 + lane];
    cnt[g] = sc[lane];
    wt[g] = sw[lane];
  }
  if (road_speed && lane == 0) {                    // lanes [0, nroad) are the road's
    const int nroad = A.tile_nroad[tile];
    double sum = 0.0;
    int c = 0;
    float vfree = 0.f;
    for (int l = 0; l < nroad; ++l) {
      sum += sv[l];
      c += sc[l];
      vfree = fmaxf(vfree, A.lane_vmax[A.tile_lanes[l0 + l]]);
    }
    road_speed[tile] = c ? (float)(sum / c) : vfree;
  }
}

__global__ void k_fill_u64(unsigned long long *p, unsigned long long v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---- partition exchange -------------------------------------------
__global__ void k_mig_header(MigRec *out_buf, const int32_t *out_off, const int32_t *out_cap,
                             int32_t *out_cnt, int world) {
  const int q = threadIdx.x;
  if (q < world) {
    if (out_cap[q] > 0) out_buf[out_off[q]].rec.vid = out_cnt[q];   // count header of region q
    out_cnt[q] = 0;                                 // ready for the next step
  }
}

// Received migrants join their tile's inbox for step t+1 exactly like local
// movers (integer atomics: order independent, so results do not depend on the
// partitioning, P-PART).  One block per peer region.
__global__ void k_absorb(StepArgs A, const MigRec *in_buf, const int32_t *in_off,
                         const int32_t *in_cap) {
  const int q = blockIdx.x;
  const int cap = in_cap[q];
  if (cap == 0) return;
  const MigRec *reg = in_buf + in_off[q];
  const int cnt = min(reg[0].rec.vid, cap);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const MigRec &m = reg[1 + i];
    const int dt = m.tile, vid = m.rec.vid;
    const int lane_g = A.tile_lanes[A.tile_lane_off[dt] + m_lane(m.rec.meta)];
    const int slot = atomicAdd(&A.icnt_out[dt], 1);
    if (slot < A.tile_icap[dt]) put_inbox(A.inbox_out + A.tile_ibase[dt] + slot, m.rec);
    atomicMin(&A.summ_next[lane_g], vkey(m.rec.s, vid));
    A.pubv_next[vid] = m.rec.v;
    if (A.lane_cnt_next) atomicAdd(&A.lane_cnt_next[lane_g], 1);
    A.insert_time[vid] = m.insert_time;
    A.status[vid] = ST_DRIVING;
  }
}

__global__ void k_halo_pack(StepArgs A, const int32_t *lanes, HaloRec *buf, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = A.summ_next[lanes[i]];
    HaloRec r;
    r.key = key;
    r.v = key != kEmptyKey ? A.pubv_next[(int)(unsigned)(key & 0xffffffffu)] : 0.f;
    r.pad = 0;
    buf[i] = r;
  }
}

__global__ void k_halo_unpack(StepArgs A, const int32_t *lanes, const HaloRec *buf, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const HaloRec r = buf[i];
    A.summ_next[lanes[i]] = r.key;
    if (r.key != kEmptyKey) A.pubv_next[(int)(unsigned)(r.key & 0xffffffffu)] = r.v;
  }
}

// ---- direct transport (NEXT-2) ------------------------------------
// Barrier over the partitions of a multi-process run: one arrival per peer
// (system-scope release after everything this stream did before), then wait
// until all `world` arrivals of this round have reached our counter.  A wait
// longer than timeout_ns (a peer died) sets *err and returns instead of hanging.
__global__ void k_barrier(const PeerView *peers, int world, int rank, unsigned target, int32_t *err,
                          unsigned long long timeout_ns) {
  const int q = threadIdx.x;
  if (q < world) {
    __threadfence_system();
    atomicAdd_system(peers[q].bar, 1u);
  }
  if (q == 0) {
    const unsigned *mine = peers[rank].bar;
    unsigned long long t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if ((int)(v - target) >= 0) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns) { atomicExch(err, 1); break; }
      __nanosleep(200);
    }
    __threadfence_system();
  }
}

// out[i] = sum over partitions q of xbuf[kind] of q at element off + i
// (dtype 0 int64, 1 int32, 2 float32; integer sums are exact, float sums of
// one non-zero contribution and zeros are exact as well).
__global__ void k_peer_sum(const PeerView *peers, int world, int kind, int dtype, int64_t off,
                           int64_t n, void *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (dtype == 0) {
      long long x = 0;
      for (int q = 0; q < world; ++q) x += reinterpret_cast<const long long *>(peers[q].xbuf[kind])[off + i];
      reinterpret_cast<long long *>(out)[i] = x;
    } else if (dtype == 1) {
      int x = 0;
      for (int q = 0; q < world; ++q) x += reinterpret_cast<const int *>(peers[q].xbuf[kind])[off + i];
      reinterpret_cast<int *>(out)[i] = x;
    } else {
      float x = 0.f;
      for (int q = 0; q < world; ++q) x += reinterpret_cast<const float *>(peers[q].xbuf[kind])[off + i];
      reinterpret_cast<float *>(out)[i] = x;
    }
  }
}

// Repartition (NEXT-2): every own tile whose new owner is
// another partition is handed over at a step boundary — its stayer rows and
// inbox records of t, its lanes' summaries / summary speeds / lane counts of
// t and pending-queue heads, and its vehicles' insert time and status are
// stored into the new owner's buffers at the same (global) positions; the old
// owner's counts for the tile become 0.  One block per own tile.
__global__ void k_rehome(StepArgs A, const int32_t *new_owner) {
  const int T = A.tiles[blockIdx.x];
  const int q = new_owner[T];
  if (q == A.rank) return;
  const PeerView &Q = A.peers[q];
  const PeerView &P = A.peers[A.rank];
  const int par = A.t & 1, s3 = A.t % 3;
  const int n = A.cnt_in[T], m = A.icnt_in[T];
  const int base = A.tile_base[T], ibase = A.tile_ibase[T];
  const Slab &D = Q.slab[par];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int g = base + i, vid = A.in.vid[g];
    D.s[g] = A.in.s[g]; D.v[g] = A.in.v[g]; D.vid[g] = vid; D.nxt[g] = A.in.nxt[g];
    D.nxt2[g] = A.in.nxt2[g]; D.meta[g] = A.in.meta[g]; D.wait[g] = A.in.wait[g];
    Q.insert_time[vid] = A.insert_time[vid];
    Q.status[vid] = ST_DRIVING;
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const InboxRec r = A.inbox_in[ibase + i];
    put_inbox(Q.inbox[par] + ibase + i, r);
    Q.insert_time[r.vid] = A.insert_time[r.vid];
    Q.status[r.vid] = ST_DRIVING;
  }
  const int l0 = A.tile_lane_off[T], nl = A.tile_lane_off[T + 1] - l0;
  for (int k = threadIdx.x; k < nl; k += blockDim.x) {
    const int g = A.tile_lanes[l0 + k];
    const unsigned long long key = A.summ_cur[g];
    Q.summ[s3][g] = key;
    Q.summ[(s3 + 1) % 3][g] = kEmptyKey;
    if (key != kEmptyKey) {
      const int vid = (int)(unsigned)(key & 0xffffffffu);
      Q.pubv[par][vid] = A.pubv_cur[vid];
    }
    if (Q.lcnt[s3] != P.lcnt[s3]) Q.lcnt[s3][g] = P.lcnt[s3][g];
    Q.pend_head[g] = A.pend_head[g];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Q.cnt[par][T] = n;
    Q.icnt[par][T] = m;
    A.cnt_in[T] = 0;
    A.icnt_in[T] = 0;
  }
}

// vehicles (stayers + inbox) of every own tile -> out[tile] (others untouched)
__global__ void k_tile_counts(StepArgs A, int32_t *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n_own; i += gridDim.x * blockDim.x) {
    const int T = A.tiles[i];
    out[T] = A.cnt_in[T] + A.icnt_in[T];
  }
}

void launch_rehome(const StepArgs &a, const int32_t *new_owner, void *stream) {
  if (a.n_own > 0) k_rehome<<<a.n_own, 128, 0, (cudaStream_t)stream>>>(a, new_owner);
}
void launch_tile_counts(const StepArgs &a, int32_t *out, void *stream) {
  if (a.n_own > 0) k_tile_counts<<<(a.n_own + 255) / 256, 256, 0, (cudaStream_t)stream>>>(a, out);
}

void launch_barrier(const PeerView *peers, int world, int rank, unsigned target, int32_t *err,
                    unsigned long long timeout_ns, void *stream) {
  k_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(peers, world, rank, target, err, timeout_ns);
}
void launch_peer_sum(const PeerView *peers, int world, int kind, int dtype, int64_t off, int64_t n,
                     void *out, void *stream) {
  if (n > 0)
    k_peer_sum<<<(int)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, (cudaStream_t)stream>>>(
        peers, world, kind, dtype, off, n, out);
}

// ---- launchers ---------------------------------------------------------------
int step_smem_bytes() { return kStepWarps * kSmemVeh * 18; }

void launch_step(const StepArgs &a, void *stream, int smem_bytes) {
  static int resident[2] = {0, 0};                  // resident blocks per GPU, per instantiation
  if (!resident[0]) {
    cudaFuncSetAttribute(k_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    int dev = 0, nsm = 0, b0 = 0, b1 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, k_step<false>, kStepWarps * kThreads, smem_bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_step<true>, kStepWarps * kThreads, smem_bytes);
    resident[0] = std::max(1, b0) * std::max(1, nsm);
    resident[1] = std::max(1, b1) * std::max(1, nsm);
  }
  if (a.n_own <= 0) return;
  const int ex = a.exact_mode ? 1 : 0;
  const int grid = std::min((a.n_own + kStepWarps - 1) / kStepWarps, resident[ex]);
  if (ex) k_step<true><<<grid, kStepWarps * kThreads, smem_bytes, (cudaStream_t)stream>>>(a);
  else k_step<false><<<grid, kStepWarps * kThreads, smem_bytes, (cudaStream_t)stream>>>(a);
}

void launch_signal(const SignalArgs &a, void *stream) {
  if (a.n_junctions > 0)
    k_signal<<<(a.n_junctions + 3) / 4, 128, 0, (cudaStream_t)stream>>>(a);
}

void launch_apply_requests(int32_t *request, uint8_t *policy, const int32_t *junc,
                           const int32_t *phase, int m, void *stream) {
  (void)policy;
  if (m > 0) k_apply_requests<<<(m + 255) / 256, 256, 0, (cudaStream_t)stream>>>(request, junc, phase, m);
}

void launch_reduce_acc(const long long *tacc, int n_tiles, const int32_t *cnt,
                       const int32_t *icnt, const uint8_t *status, int nv, long long *out,
                       void *stream) {
  cudaMemsetAsync(out, 0, (kNAcc + 3) * sizeof(long long), (cudaStream_t)stream);
  k_reduce_acc<<<296, 256, 0, (cudaStream_t)stream>>>(tacc, n_tiles, cnt, icnt, status, nv, out);
}

void launch_lane_stats(const StepArgs &a, int32_t *lane_count, int32_t *lane_wait,
                       float *road_speed, float zone, void *stream) {
  if (a.n_own > 0)
    k_lane_stats<<<(a.n_own + 3) / 4, 128, 0, (cudaStream_t)stream>>>(a, lane_count, lane_wait, road_speed, zone);
}

void launch_reduce_groups(const long long *tacc, const int32_t *tiles, int n_own,
                          const int32_t *tile_group, const int32_t *cnt, const int32_t *icnt,
                          int n_groups, long long *out, void *stream) {
  cudaMemsetAsync(out, 0, (size_t)n_groups * (kNAcc + 1) * sizeof(long long), (cudaStream_t)stream);
  if (n_own > 0)
    k_reduce_groups<<<296, 256, 0, (cudaStream_t)stream>>>(tacc, tiles, n_own, tile_group, cnt, icnt, out);
}

// set_vehicle_route: every DRIVING vehicle with patch[vid] >= 0
// restarts at cursor patch[vid] (0) of its new route; its cached next roads
// are refreshed in the slab or inbox record that holds it.
__global__ void k_patch_routes(StepArgs A, const int32_t *patch) {
  const int tile = A.tiles[blockIdx.x];
  const int ns = A.cnt_in[tile], ni = A.icnt_in[tile];
  for (int i = threadIdx.x; i < ns + ni; i += blockDim.x) {
    int vid;
    uint32_t *meta;
    int32_t *nxt, *nxt2;
    InboxRec *r = nullptr;
    if (i < ns) {
      const int gi = A.tile_base[tile] + i;
      vid = A.in.vid[gi]; meta = A.in.meta + gi; nxt = A.in.nxt + gi; nxt2 = A.in.nxt2 + gi;
    } else {
      r = const_cast<InboxRec *>(A.inbox_in) + A.tile_ibase[tile] + i - ns;
      vid = r->vid; meta = &r->meta; nxt = &r->nxt; nxt2 = &r->nxt2;
    }
    const int c = patch[vid];
    if (c < 0) continue;
    const int off = A.route_start[vid], len = A.route_len[vid];
    *meta = (*meta & 0xffffu) | ((uint32_t)c << 16);
    *nxt = c + 1 < len ? A.route[off + c + 1] : -1;
    *nxt2 = c + 2 < len ? A.route[off + c + 2] : -1;
  }
}

// set_vehicle_route support: where is each vehicle of a batch (want[vid] =
// batch index b)?  out[2b] = cursor, out[2b+1] = global lane (DRIVING only).
__global__ void k_locate(StepArgs A, const int32_t *want, int32_t *out) {
  const int tile = A.tiles[blockIdx.x];
  const int ns = A.cnt_in[tile], ni = A.icnt_in[tile];
  const int l0 = A.tile_lane_off[tile];
  for (int i = threadIdx.x; i < ns + ni; i += blockDim.x) {
    int vid;
    uint32_t meta;
    if (i < ns) {
      const int gi = A.tile_base[tile] + i;
      vid = A.in.vid[gi]; meta = A.in.meta[gi];
    } else {
      const InboxRec &r = A.inbox_in[A.tile_ibase[tile] + i - ns];
      vid = r.vid; meta = r.meta;
    }
    const int b = want[vid];
    if (b < 0) continue;
    out[2 * b] = m_cursor(meta);
    out[2 * b + 1] = A.tile_lanes[l0 + m_lane(meta)];
  }
}

__global__ void k_scatter_i32(int32_t *dst, const int32_t *idx, const int32_t *val, int32_t cval,
                              int m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) dst[idx[i]] = val ? val[i] : cval;
}
__global__ void k_scatter_f32(float *dst, const int32_t *idx, const float *val, int m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) dst[idx[i]] = val[i];
}

__global__ void k_gather_u8(const uint8_t *src, const int32_t *idx, uint8_t *out, int m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = src[idx[i]];
}
void launch_gather_u8(const uint8_t *src, const int32_t *idx, uint8_t *out, int m, void *stream) {
  if (m > 0) k_gather_u8<<<(m + 255) / 256, 256, 0, (cudaStream_t)stream>>>(src, idx, out, m);
}

void launch_locate(const StepArgs &a, const int32_t *want, int32_t *out, void *stream) {
  if (a.n_own > 0) k_locate<<<a.n_own, 128, 0, (cudaStream_t)stream>>>(a, want, out);
}
void launch_scatter_i32(int32_t *dst, const int32_t *idx, const int32_t *val, int32_t cval, int m,
                        void *stream) {
  if (m > 0) k_scatter_i32<<<(m + 255) / 256, 256, 0, (cudaStream_t)stream>>>(dst, idx, val, cval, m);
}
void launch_scatter_f32(float *dst, const int32_t *idx, const float *val, int m, void *stream) {
  if (m > 0) k_scatter_f32<<<(m + 255) / 256, 256, 0, (cudaStream_t)stream>>>(dst, idx, val, m);
}

void launch_patch_routes(const StepArgs &a, const int32_t *patch, void *stream) {
  if (a.n_own > 0) k_patch_routes<<<a.n_own, 128, 0, (cudaStream_t)stream>>>(a, patch);
}

void launch_fill_u64(unsigned long long *p, unsigned long long v, int64_t n, void *stream) {
  if (n > 0) k_fill_u64<<<256, 256, 0, (cudaStream_t)stream>>>(p, v, n);
}

void launch_set_i32(int32_t *, const int32_t *, const int32_t *, int, void *) {}

void launch_mig_header(MigRec *out_buf, const int32_t *out_off, const int32_t *out_cap,
                       int32_t *out_cnt, int world, void *stream) {
  k_mig_header<<<1, 32, 0, (cudaStream_t)stream>>>(out_buf, out_off, out_cap, out_cnt, world);
}
void launch_absorb(const StepArgs &a, const MigRec *in_buf, const int32_t *in_off,
                   const int32_t *in_cap, int world, void *stream) {
  k_absorb<<<world, 256, 0, (cudaStream_t)stream>>>(a, in_buf, in_off, in_cap);
}
void launch_halo_pack(const StepArgs &a, const int32_t *lanes, HaloRec *buf, int64_t n, void *stream) {
  if (n > 0) k_halo_pack<<<(int)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, (cudaStream_t)stream>>>(a, lanes, buf, n);
}
void launch_halo_unpack(const StepArgs &a, const int32_t *lanes, const HaloRec *buf, int64_t n,
                        void *stream) {
  if (n > 0) k_halo_unpack<<<(int)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, (cudaStream_t)stream>>>(a, lanes, buf, n);
}

}  // namespace sim

extern "C" int sim_debug_guard_stats(unsigned long long *out) {
#ifdef GUARD_STATS
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, sim::g_guard_stats, 32 * 8) == cudaSuccess ? 32 : -1;
#else
  (void)out;
  return 0;
#endif
}

namespace sim {

}  // namespace sim
