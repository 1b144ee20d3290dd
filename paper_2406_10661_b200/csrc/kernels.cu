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
#ifndef F64_NOINLINE
#define F64_NOINLINE __forceinline__
#endif
#ifdef GUARD_STATS
__device__ unsigned long long g_guard_stats[32];
#endif
__device__ F64_NOINLINE void veh_update_f64(const StepArgs &A, const TileSh &T, const View &C,
                                            int i, Res &r) {
  Guard g;
  g.hit = false;
  g.why = 0;
  veh_update<double, false>(A, T, C, i, r, g);
}

struct ResView {                     // per-slot step results (shared or global scratch)
  float *s1, *v1;
  int32_t *lane, *wait, *cur;
  uint8_t *flags;                    // lc+1 : 2 | fin : 1 | min(hand, 31) : 5
};
__device__ __forceinline__ void store_res(const ResView &R, int i, const Res &r) {
  R.s1[i] = r.s1;
  R.v1[i] = r.v1;
  R.lane[i] = r.lane_g;
  R.wait[i] = r.wait1;
  R.cur[i] = r.cursor;
  R.flags[i] = (uint8_t)((r.lc + 1) | (r.fin ? 4 : 0) | ((r.hand > 31 ? 31 : r.hand) << 3));
}
__device__ __forceinline__ void load_res(const ResView &R, int i, Res &r) {
  r.s1 = R.s1[i];
  r.v1 = R.v1[i];
  r.lane_g = R.lane[i];
  r.wait1 = R.wait[i];
  r.cursor = R.cur[i];
  const int f = R.flags[i];
  r.lc = (f & 3) - 1;
  r.fin = (f & 4) != 0;
  r.hand = f >> 3;
}
__device__ __forceinline__ void record(const StepArgs &A, int vid, const Res &r, bool guard) {
  A.r_leader[vid] = r.leader;
  A.r_hops[vid] = (int8_t)r.hops;
  A.r_phantom[vid] = (int8_t)r.phantom;
  A.r_of[vid] = r.of_vid;
  for (int q = 0; q < 4; ++q) A.r_side[4 * vid + q] = r.side[q];
  A.r_lc[vid] = (int8_t)r.lc;
  A.r_hand[vid] = (int8_t)(r.hand > 127 ? 127 : r.hand);
  A.r_acc[vid] = r.acc;
  A.r_fin[vid] = (int8_t)r.fin;
  A.r_guard[vid] = (uint8_t)(guard ? 1 : 0);
}

struct StepShared {
  TileSh T;
  int warp_tot[kThreads / 32];
  int nst_out;
  int nguard;
  unsigned long long bk_hi[kSmemInbox];
  int bk_vid[kSmemInbox];
  int bsort[kSmemInbox];
  unsigned long long sk_hi[kSmemInbox];   // inbox keys in sorted order
  int sk_vid[kSmemInbox];
  Prof prof[kSmemProf];
  long long acc[kNAcc];
};

#ifndef KSTEP_MINB
#define KSTEP_MINB 8
#endif
__global__ void __launch_bounds__(kThreads, KSTEP_MINB) k_step(StepArgs A) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ StepShared S;
  TileSh &T = S.T;
  const int tile = blockIdx.x, tid = threadIdx.x;
  const int lane_id = tid & 31, warp = tid >> 5;

  // ---- tile metadata -----------------------------------------------------
  const int l0 = A.tile_lane_off[tile];
  const int nl = A.tile_lane_off[tile + 1] - l0;
  if (tid == 0) {
    T.nl = nl;
    T.nroad = A.tile_nroad[tile];
    T.tile = tile;
    T.base = A.tile_base[tile];
    T.ibase = A.tile_ibase[tile];
    T.cap = A.tile_cap[tile];
    T.icap = A.tile_icap[tile];
    S.nst_out = 0;
    S.nguard = 0;
    T.P = A.n_prof <= kSmemProf ? S.prof : A.prof;
  }
  if (tid < kNAcc) S.acc[tid] = 0;
  if (A.n_prof <= kSmemProf)
    for (int q = tid; q < A.n_prof; q += kThreads) S.prof[q] = A.prof[q];
  for (int l = tid; l < nl; l += kThreads) {
    int g = A.tile_lanes[l0 + l];
    T.glob[l] = g;
    T.len[l] = A.lane_len[g];
    T.vmax[l] = A.lane_vmax[g];
    T.isroad[l] = A.lane_road[g] >= 0;
    T.usable[l] = A.usable[g];
    T.seg_start[l] = 0;
    T.seg_end[l] = 0;
    T.first_out[l] = 0x7fffffff;
    int lf = A.lane_left ? A.lane_left[g] : -1, rt = A.lane_right ? A.lane_right[g] : -1;
    T.left[l] = (lf >= 0 && A.lane_tile[lf] == tile) ? (int8_t)A.lane_local[lf] : (int8_t)-1;
    T.right[l] = (rt >= 0 && A.lane_tile[rt] == tile) ? (int8_t)A.lane_local[rt] : (int8_t)-1;
  }
  // successor table of the tile's road lanes (usable successors only)
  const int nroad = A.tile_nroad[tile];
  if (tid == 0) T.tab_ok = nroad <= kMaxRoadLanes ? 1 : 0;
  if (nroad <= kMaxRoadLanes) {
    for (int l = tid; l < nroad; l += kThreads) {
      const int g = A.tile_lanes[l0 + l];
      const int e0 = A.succ_off[g], e1 = A.succ_off[g + 1];
      int k = 0;
      bool ok = e1 - e0 <= kMaxSucc;
      if (ok)
        for (int e = e0; e < e1; ++e) {
          const int j = A.succ[e];
          if (!A.usable[j]) continue;
          SuccEnt &s = T.se[l][k++];
          s.j = j;
          s.troad = A.target_road[j];
          s.b = A.exit_lane[j];
          s.outr = A.outroads[s.b];
          s.stop = (A.lane_road[j] < 0 && A.lane_sig[j] != SIG_GREEN) ? 1 : 0;
        }
      T.sn[l] = (uint8_t)k;
      if (!ok) T.tab_ok = 0;
    }
  }
  const int n_st = A.cnt_in[tile];
  const int n_in = A.icnt_in[tile];
  const int n = n_st + n_in;
  const int base = A.tile_base[tile];
  const int ibase = A.tile_ibase[tile];

  // snapshot view: shared memory, or this tile's global scratch if too large
  View C;
  const bool smem_ok = (n <= kSmemVeh) && (n_in <= kSmemInbox);
  if (smem_ok) {
    float *f = reinterpret_cast<float *>(dyn);
    C.s = f;
    C.v = f + kSmemVeh;
    C.vid = reinterpret_cast<int32_t *>(f + 2 * kSmemVeh);
    C.nxt = C.vid + kSmemVeh;
    C.nxt2 = C.vid + 2 * kSmemVeh;
    C.meta = reinterpret_cast<uint32_t *>(C.vid + 3 * kSmemVeh);
    C.wait = C.vid + 4 * kSmemVeh;
  } else {
    const int sb = base + ibase;               // scratch is indexed by base + ibase (size cap + icap)
    C.s = A.scratch.s + sb;
    C.v = A.scratch.v + sb;
    C.vid = A.scratch.vid + sb;
    C.nxt = A.scratch.nxt + sb;
    C.nxt2 = A.scratch.nxt2 + sb;
    C.meta = A.scratch.meta + sb;
    C.wait = A.scratch.wait + sb;
  }
  int *bsort = (n_in <= kSmemInbox) ? S.bsort : (A.bsort_scratch + ibase);
  const InboxRec *inb = A.inbox_in + ibase;

  // ---- 1. merge stayers + sorted inbox (a1) ---------------------------------
  if (n_in > 0) {
    if (n_in <= kSmemInbox) {
      for (int j = tid; j < n_in; j += kThreads) {
        InboxRec r = inb[j];
        S.bk_hi[j] = hikey(m_lane(r.meta), r.s);
        S.bk_vid[j] = r.vid;
      }
      __syncthreads();
      for (int j = tid; j < n_in; j += kThreads) {
        unsigned long long h = S.bk_hi[j];
        int vj = S.bk_vid[j], rank = 0;
        for (int q = 0; q < n_in; ++q) rank += key_less(S.bk_hi[q], S.bk_vid[q], h, vj);
        bsort[rank] = j;
        S.sk_hi[rank] = h;
        S.sk_vid[rank] = vj;
      }
    } else {
      for (int j = tid; j < n_in; j += kThreads) {
        InboxRec r = inb[j];
        unsigned long long h = hikey(m_lane(r.meta), r.s);
        int rank = 0;
        for (int q = 0; q < n_in; ++q) {
          InboxRec o = inb[q];
          rank += key_less(hikey(m_lane(o.meta), o.s), o.vid, h, r.vid);
        }
        bsort[rank] = j;
      }
    }
  }
  __syncthreads();
  // stayers: position = own index + #inbox keys below (binary search in sorted inbox)
  for (int i = tid; i < n_st; i += kThreads) {
    const int gi = base + i;
    float s = A.in.s[gi];
    uint32_t meta = A.in.meta[gi];
    int vid = A.in.vid[gi];
    int pos = i;
    if (n_in > 0) {
      unsigned long long h = hikey(m_lane(meta), s);
      int lo = 0, hi = n_in;
      if (n_in <= kSmemInbox) {
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (key_less(S.sk_hi[mid], S.sk_vid[mid], h, vid)) lo = mid + 1; else hi = mid;
        }
      } else {
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          InboxRec o = inb[bsort[mid]];
          if (key_less(hikey(m_lane(o.meta), o.s), o.vid, h, vid)) lo = mid + 1; else hi = mid;
        }
      }
      pos += lo;
    }
    C.s[pos] = s;
    C.v[pos] = A.in.v[gi];
    C.vid[pos] = vid;
    C.nxt[pos] = A.in.nxt[gi];
    C.nxt2[pos] = A.in.nxt2[gi];
    C.meta[pos] = meta;
    C.wait[pos] = A.in.wait[gi];
  }
  // inbox records: position = sorted rank + #stayers below (binary search in slab)
  for (int r = tid; r < n_in; r += kThreads) {
    InboxRec rec = inb[bsort[r]];
    unsigned long long h = hikey(m_lane(rec.meta), rec.s);
    int lo = 0, hi = n_st;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      int gi = base + mid;
      if (key_less(hikey(m_lane(A.in.meta[gi]), A.in.s[gi]), A.in.vid[gi], h, rec.vid)) lo = mid + 1;
      else hi = mid;
    }
    int pos = r + lo;
    C.s[pos] = rec.s;
    C.v[pos] = rec.v;
    C.vid[pos] = rec.vid;
    C.nxt[pos] = rec.nxt;
    C.nxt2[pos] = rec.nxt2;
    C.meta[pos] = rec.meta;
    C.wait[pos] = rec.wait;
  }
  __syncthreads();
  // lane segments of the snapshot
  for (int i = tid; i < n; i += kThreads) {
    int l = m_lane(C.meta[i]);
    if (i == 0 || m_lane(C.meta[i - 1]) != l) T.seg_start[l] = i;
    if (i == n - 1 || m_lane(C.meta[i + 1]) != l) T.seg_end[l] = i + 1;
  }
  __syncthreads();

  // ---- 2. per-vehicle update (a2-a4), results staged per snapshot slot ------
  // Phase A: every vehicle on the fp32 fast path; vehicles whose decision
  // margins fall inside the guard band are queued.  Phase B: the queue is
  // recomputed with the canonical fp64 sequence, packed onto few lanes (so a
  // rare fallback does not stall whole warps).  No barrier inside either loop.
  ResView R;
  int *glist;
  if (smem_ok) {
    unsigned char *rb = dyn + kSmemVeh * 7 * 4;
    R.s1 = reinterpret_cast<float *>(rb);
    R.v1 = R.s1 + kSmemVeh;
    R.lane = reinterpret_cast<int32_t *>(R.v1 + kSmemVeh);
    R.wait = R.lane + kSmemVeh;
    R.cur = R.wait + kSmemVeh;
    glist = R.cur + kSmemVeh;
    R.flags = reinterpret_cast<uint8_t *>(glist + kSmemVeh);
  } else {
    const int sb = base + ibase;
    R.s1 = A.rs_s1 + sb;
    R.v1 = A.rs_v1 + sb;
    R.lane = A.rs_lane + sb;
    R.wait = A.rs_wait + sb;
    R.cur = A.rs_cur + sb;
    R.flags = A.rs_flags + sb;
    glist = A.rs_glist + sb;
  }
  long long acc_travel = 0, acc_waitfin = 0;
  int acc_fin = 0, acc_lc = 0, acc_hand = 0, acc_guard = 0, acc_ovf = 0;
  for (int i = tid; i < n; i += kThreads) {
    Res r;
    Guard g;
    g.hit = false;
    g.why = 0;
    if (A.exact_mode) {
      veh_update_f64(A, T, C, i, r);
    } else {
      veh_update<float, true>(A, T, C, i, r, g);
      if (g.hit) {
        glist[atomicAdd(&S.nguard, 1)] = i;
        acc_guard += 1;
#ifdef GUARD_STATS
        for (int b = 0; b < 32; ++b)
          if (g.why & (1u << b)) atomicAdd(&g_guard_stats[b], 1ull);
#endif
      }
    }
    store_res(R, i, r);
    if (A.record) record(A, C.vid[i], r, g.hit);
  }
  __syncthreads();
  for (int q = tid; q < S.nguard; q += kThreads) {
    const int i = glist[q];
    Res r;
    veh_update_f64(A, T, C, i, r);
    store_res(R, i, r);
    if (A.record) record(A, C.vid[i], r, true);
  }
  __syncthreads();

  // ---- 3. outputs, in chunks of kThreads (order-preserving compaction) -------
  const int nchunks = (n + kThreads - 1) / kThreads;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int i = ch * kThreads + tid;
    int kind = 0;                      // 0 none, 1 stayer, 2 mover, 3 finished
    Res r;
    if (i < n) {
      load_res(R, i, r);
      const int l = m_lane(C.meta[i]);
      if (r.fin) kind = 3;
      else if (r.lc == 0 && r.hand == 0 && r.lane_g == T.glob[l]) kind = 1;
      else kind = 2;
    }
    // order-preserving compaction of stayers (block scan)
    const unsigned ball = __ballot_sync(0xffffffffu, kind == 1);
    const int wprefix = __popc(ball & ((1u << lane_id) - 1u));
    if (lane_id == 0) S.warp_tot[warp] = __popc(ball);
    __syncthreads();
    int woff = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const int x = S.warp_tot[w];
      woff += (w < warp) ? x : 0;
      tot += x;
    }
    const int run = S.nst_out;
    if (kind == 1) {
      const int pos = base + run + woff + wprefix;
      const uint32_t meta = C.meta[i];
      A.out.s[pos] = r.s1;
      A.out.v[pos] = r.v1;
      A.out.vid[pos] = C.vid[i];
      A.out.nxt[pos] = C.nxt[i];
      A.out.nxt2[pos] = C.nxt2[i];
      A.out.meta[pos] = meta;
      A.out.wait[pos] = r.wait1;
      atomicMin(&T.first_out[m_lane(meta)], pos);
    } else if (kind == 2) {
      const int vid = C.vid[i];
      const uint32_t meta = C.meta[i];
      const int cur = m_cursor(meta);
      InboxRec rec;
      rec.s = r.s1;
      rec.v = r.v1;
      rec.vid = vid;
      rec.nxt = route_at(A, vid, cur, C.nxt[i], C.nxt2[i], r.cursor + 1);
      rec.nxt2 = route_at(A, vid, cur, C.nxt[i], C.nxt2[i], r.cursor + 2);
      rec.meta = pack_meta(A.lane_local[r.lane_g], m_prof(meta), r.cursor);
      rec.wait = r.wait1;
      rec.pad = 0;
      const int dt = A.lane_tile[r.lane_g];
      const int slot = atomicAdd(&A.icnt_out[dt], 1);
      if (slot < A.tile_icap[dt]) {
        int4 *dst = reinterpret_cast<int4 *>(A.inbox_out + A.tile_ibase[dt] + slot);
        const int4 *src = reinterpret_cast<const int4 *>(&rec);
        dst[0] = src[0];
        dst[1] = src[1];
      } else {
        acc_ovf += 1;
      }
      atomicMin(&A.summ_next[r.lane_g], vkey(r.s1, vid));
      A.pubv_next[vid] = r.v1;
      acc_lc += r.lc != 0;
      acc_hand += r.hand;
    } else if (kind == 3) {
      const int vid = C.vid[i];
      A.status[vid] = ST_FINISHED;
      A.arrive_time[vid] = A.t + 1;
      A.wait_fin[vid] = r.wait1;
      acc_fin += 1;
      acc_travel += (long long)(A.t + 1 - A.insert_time[vid]);
      acc_waitfin += r.wait1;
      acc_lc += r.lc != 0;
      acc_hand += r.hand;
    }
    __syncthreads();
    if (tid == 0) S.nst_out = run + tot;
    __syncthreads();
  }

  // ---- 4. summaries, insertions, counters ------------------------------------
  for (int l = tid; l < nl; l += kThreads) {
    const int g = T.glob[l];
    const int pos = T.first_out[l];
    if (pos != 0x7fffffff) {
      const float s1 = A.out.s[pos];
      const int vid = A.out.vid[pos];
      atomicMin(&A.summ_next[g], vkey(s1, vid));
      A.pubv_next[vid] = A.out.v[pos];
    }
    A.summ_clear[g] = kEmptyKey;
  }
  int acc_ins = 0;
  long long acc_delay = 0;
  for (int l = tid; l < T.nroad; l += kThreads) {   // departures (K11; ledger L25)
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
      const double sa = C.s[fa], la = T.P[m_prof(C.meta[fa])].len_d;
      if (!(__dadd_rn(__dadd_rn(sa, -ss), -la) >= pk.s0_d)) ok = false;
    }
    if (fa > a0) {
      const int b = fa - 1;
      const Prof &pb = T.P[m_prof(C.meta[b])];
      const double need = __dadd_rn(__dadd_rn((double)C.v[b], __dmul_rn(0.5, pb.a_max_d)), pk.s0_d);
      if (!(__dadd_rn(__dadd_rn(ss, -(double)C.s[b]), -pk.len_d) >= need)) ok = false;
    } else {
      if (!(__dadd_rn(ss, -pk.len_d) >= A.start_margin)) ok = false;
    }
    if (!ok) continue;
    InboxRec rec;
    rec.s = (float)ss;
    rec.v = 0.f;
    rec.vid = k;
    const int off = A.route_off[k], rl = A.route_off[k + 1] - off;
    rec.nxt = rl > 1 ? A.route[off + 1] : -1;
    rec.nxt2 = rl > 2 ? A.route[off + 2] : -1;
    rec.meta = pack_meta(l, A.veh_prof[k], 0);
    rec.wait = 0;
    rec.pad = 0;
    const int slot = atomicAdd(&A.icnt_out[tile], 1);
    if (slot < T.icap) {
      int4 *dst = reinterpret_cast<int4 *>(A.inbox_out + ibase + slot);
      const int4 *src = reinterpret_cast<const int4 *>(&rec);
      dst[0] = src[0];
      dst[1] = src[1];
    } else {
      acc_ovf += 1;
    }
    atomicMin(&A.summ_next[g], vkey(rec.s, k));
    A.pubv_next[k] = 0.f;
    A.pend_head[g] = h + 1;
    A.status[k] = ST_DRIVING;
    A.insert_time[k] = A.t + 1;
    if (A.record) A.r_ins[k] = 1;
    acc_ins += 1;
    acc_delay += (long long)(A.t + 1 - A.depart[k]);
  }
  // block reduction of the counters (int64 shared atomics, exact, order independent)
  const long long vals[kNAcc] = {0, acc_fin, acc_travel, acc_waitfin, acc_delay, acc_lc, acc_hand,
                                 acc_ins, acc_guard, acc_ovf, 0, 0};
#pragma unroll
  for (int c = 1; c < kNAcc; ++c)
    if (vals[c]) atomicAdd(reinterpret_cast<unsigned long long *>(&S.acc[c]),
                           (unsigned long long)vals[c]);
  __syncthreads();
  if (tid == 0) {
    long long *ta = A.tacc + (size_t)tile * kNAcc;
    ta[ACC_VEH_STEPS] += n;
    for (int c = 1; c < kNAcc; ++c) ta[c] += S.acc[c];
    A.cnt_out[tile] = S.nst_out;
    A.icnt_in[tile] = 0;
  }
}

// ---- a5: per-junction signal controller -------------
__global__ void k_signal(SignalArgs a) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n_junctions) return;
  const int K = a.ph_off[j + 1] - a.ph_off[j];
  int pol = a.policy[j], ph = a.phase[j], el = a.elapsed[j], y = a.yellow_left[j],
      q = a.pending[j];
  const int req = a.request[j];
  if (req >= 0) {                                   // requests apply before sig_t (L35)
    a.request[j] = -1;
    pol = POL_MANUAL;
    if (y > 0) q = req;
    else if (req != ph) {
      if (a.yellow > 0) { y = a.yellow; q = req; }
      else { ph = req; q = req; }
    }
  }
  const int j0 = a.jl_off[j], nj = a.jl_off[j + 1] - j0;
  const uint8_t *grow = a.green + a.green_off[j] + (int64_t)ph * nj;
  for (int k = 0; k < nj; ++k) {
    uint8_t sg;
    if (pol == POL_NONE || K == 0) sg = SIG_GREEN;
    else {
      const bool g = grow[k] != 0;
      sg = y > 0 ? (g ? SIG_YELLOW : SIG_RED) : (g ? SIG_GREEN : SIG_RED);
    }
    a.lane_sig[a.jl[j0 + k]] = sg;
  }
  // advance t -> t+1 (O11)
  if (pol == POL_FIXED && K > 0) {
    if (y > 0) {
      y -= 1;
      if (y == 0) { ph = q; el = 0; }
    } else {
      el += 1;
      if (el >= a.green_steps[a.ph_off[j] + ph]) {
        const int nx = (ph + 1) % K;
        if (a.yellow > 0) { y = a.yellow; q = nx; }
        else { ph = nx; q = nx; el = 0; }
      }
    }
  } else if (pol == POL_MANUAL) {
    if (y > 0) {
      y -= 1;
      if (y == 0) ph = q;
    }
    el += 1;
  }
  a.policy[j] = (uint8_t)pol;
  a.phase[j] = ph;
  a.elapsed[j] = el;
  a.yellow_left[j] = y;
  a.pending[j] = q;
}

__global__ void k_apply_requests(int32_t *request, uint8_t *policy, const int32_t *junc,
                                 const int32_t *phase, int m) {
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int i = 0; i < m; ++i) request[junc[i]] = phase[i];   // in order
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

__global__ void k_lane_stats(StepArgs A, int32_t *cnt, int32_t *wt, float zone) {
  // lane queue length: per lane, vehicles and those with v < v_wait
  // within the last `zone` metres, over stayers + inbox of each tile
  const int tile = blockIdx.x;
  const int ns = A.cnt_in[tile], ni = A.icnt_in[tile];
  const int l0 = A.tile_lane_off[tile];
  for (int i = threadIdx.x; i < ns + ni; i += blockDim.x) {
    float s, v;
    uint32_t meta;
    if (i < ns) {
      const int gi = A.tile_base[tile] + i;
      s = A.in.s[gi]; v = A.in.v[gi]; meta = A.in.meta[gi];
    } else {
      const InboxRec r = A.inbox_in[A.tile_ibase[tile] + i - ns];
      s = r.s; v = r.v; meta = r.meta;
    }
    const int g = A.tile_lanes[l0 + m_lane(meta)];
    atomicAdd(&cnt[g], 1);
    if (v < A.v_wait && (A.lane_len[g] - s) <= zone) atomicAdd(&wt[g], 1);
  }
}

__global__ void k_fill_u64(unsigned long long *p, unsigned long long v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---- launchers ---------------------------------------------------------------
int step_smem_bytes() { return kSmemVeh * (7 * 4 + 6 * 4 + 1); }

void launch_step(const StepArgs &a, void *stream, int smem_bytes) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    attr = true;
  }
  if (a.n_tiles > 0)
    k_step<<<a.n_tiles, kThreads, smem_bytes, (cudaStream_t)stream>>>(a);
}

void launch_signal(const SignalArgs &a, void *stream) {
  if (a.n_junctions > 0)
    k_signal<<<(a.n_junctions + 127) / 128, 128, 0, (cudaStream_t)stream>>>(a);
}

void launch_apply_requests(int32_t *request, uint8_t *policy, const int32_t *junc,
                           const int32_t *phase, int m, void *stream) {
  k_apply_requests<<<1, 1, 0, (cudaStream_t)stream>>>(request, policy, junc, phase, m);
}

void launch_reduce_acc(const long long *tacc, int n_tiles, const int32_t *cnt,
                       const int32_t *icnt, const uint8_t *status, int nv, long long *out,
                       void *stream) {
  cudaMemsetAsync(out, 0, (kNAcc + 3) * sizeof(long long), (cudaStream_t)stream);
  k_reduce_acc<<<296, 256, 0, (cudaStream_t)stream>>>(tacc, n_tiles, cnt, icnt, status, nv, out);
}

void launch_lane_stats(const StepArgs &a, int32_t *lane_count, int32_t *lane_wait, float zone,
                       void *stream) {
  if (a.n_tiles > 0)
    k_lane_stats<<<a.n_tiles, 128, 0, (cudaStream_t)stream>>>(a, lane_count, lane_wait, zone);
}

void launch_fill_u64(unsigned long long *p, unsigned long long v, int64_t n, void *stream) {
  if (n > 0) k_fill_u64<<<256, 256, 0, (cudaStream_t)stream>>>(p, v, n);
}

void launch_set_i32(int32_t *, const int32_t *, const int32_t *, int, void *) {}

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
