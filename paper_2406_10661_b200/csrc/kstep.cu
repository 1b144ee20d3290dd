// kstep.cu — the step kernel k_step_w (rows a0-a4, a6) and k_prep.
//
// k_step_w: one warp per CTA, 16 CTAs per SM, persistent.  Each warp claims a
// tile (a road's lanes + the junction lanes leaving it, dev.h) from a global
// counter in an order k_prep builds (largest estimated work first),
// bulk-copies the tile's block — descriptor + what k_prep staged from other
// tiles: the first vehicle of every junction lane's exit lane at t (the
// P:168-169 lookahead target), the junction lanes' signals, the heads of the
// pending-departure queues — into its own shared area (cp.async.bulk +
// mbarrier), merges the tile's in-order stayers and its inbox from global
// memory into a shared snapshot (a1), runs the fused
// per-vehicle update (eligibility, leader / lookahead, IDM, MOBIL, integrate,
// hand-off, arrival: a2-a4), recomputes the vehicles whose fp32
// margins fell inside the guard band on the canonical fp64 path,
// and compacts the stayers / writes the lane summaries for t+1 / inserts
// departures (K11) / adds the counters (a6).  Tiles too large for the
// area run whole in global mode (snapshot and pass state in global scratch,
// passes 1-3 below).  (The warp-specialised ring kernel of earlier in round 2
// — producer warp + consumer rounds — is in git history.)
//
// Every decision reads only state(t) (the snapshot) and all
// cross-tile outputs are integer atomics into the t+1 buffers, so the result
// does not depend on which CTA or warp takes which tile or in what order.
#include <cuda_runtime.h>

#include <algorithm>

#include "dev.h"
#include "model.cuh"

namespace sim {

#ifndef KW_ORDER
#define KW_ORDER 2                                  // k_step_w tile order: 1 vehicles, 2 vehicles + 4 x lanes (k_prep buckets)
#endif
#ifndef KW_BSHIFT
#define KW_BSHIFT kBucketShift
#endif
// Byte layout of a tile's slot in global mode (run_tile<EXACT, true>): only
// the block (descriptor + the k_prep staging) at offset 0; the snapshot and
// the pass state live in the global scratch arrays.
struct SlotLayout {
  uint32_t veh, desc, snap, sortk, size;
  int n4;
};
__device__ __forceinline__ SlotLayout slot_layout(int n_st, int n_in, int dw) {
  SlotLayout L;
  L.n4 = (n_st + n_in + 3) & ~3;
  uint32_t o = 0;
  L.veh = o;   o += 32u * (uint32_t)L.n4;              // InboxRec records, then the PState
  L.desc = o;  o += 4u * (uint32_t)dw;                 // dw is a multiple of 4
  L.snap = o;  o += 32u * (uint32_t)L.n4;              // merged snapshot (View, stride n4)
  L.sortk = o; o += 16u * (uint32_t)n_in;              // sorted inbox keys
  L.size = o;
  return L;
}

struct __align__(16) Hdr {          // a tile's fields (from its static record and counts)
  int tile, n_st, n_in, base, ibase, cap, icap, nl, nroad, dw, dwd;
  int gm, done;                     // global mode / end-of-work sentinel
  uint32_t off;                     // slot byte offset in the ring
};

// per-vehicle pass state of one tile (slot in shared memory, or the global
// pass scratch for a tile in global mode), indexed by snapshot position;
// 30 B per vehicle (fits the 32 B of the vehicle record it replaces).  The
// stayer results rs1 / rv1 share pa / plim: both are written by the thread
// that has just read a / lim of the same vehicle (pass 3, fp64 path).
struct PState {
  unsigned char *p;                  // base of the tile's pass state
  int n4;                            // stride (slots, multiple of 4)
  __device__ __forceinline__ float &pa(int i) const { return reinterpret_cast<float *>(p)[i]; }
  __device__ __forceinline__ float &plim(int i) const { return reinterpret_cast<float *>(p)[n4 + i]; }
  __device__ __forceinline__ float &plimrel(int i) const { return reinterpret_cast<float *>(p)[2 * n4 + i]; }
  __device__ __forceinline__ float &pvlim(int i) const { return reinterpret_cast<float *>(p)[3 * n4 + i]; }
  __device__ __forceinline__ float &rs1(int i) const { return pa(i); }
  __device__ __forceinline__ float &rv1(int i) const { return plim(i); }
  __device__ __forceinline__ int &pnext1(int i) const { return reinterpret_cast<int *>(p)[4 * n4 + i]; }
  __device__ __forceinline__ uint32_t &pfl(int i) const { return reinterpret_cast<uint32_t *>(p)[5 * n4 + i]; }
  __device__ __forceinline__ uint8_t &kind(int i) const { return p[24 * n4 + i]; }
  __device__ __forceinline__ uint16_t *cand() const { return reinterpret_cast<uint16_t *>(p + 25 * n4); }
  __device__ __forceinline__ uint16_t *defl() const { return reinterpret_cast<uint16_t *>(p + 27 * n4); }
  __device__ __forceinline__ uint8_t &pnl(int i) const { return p[29 * n4 + i]; }
};
__device__ __forceinline__ PState pstate_at(unsigned char *p, int n4) {
  PState S;
  S.p = p;
  S.n4 = n4;
  return S;
}

#ifdef KS_NOGUARD
constexpr bool kGuard = false;                // timing experiment only (no fp64 fallback)
#else
constexpr bool kGuard = true;
#endif

// pass-state flag bits
enum : uint32_t {
  F_LIM = 1u, F_HIT = 2u, F_ING = 4u, F_W0 = 8u, F_W1 = 16u,
  F_MAND_SH = 5,                    // 2 bits: mand + 1
  F_K_SH = 8,                       // 5 bits: troad index + 1
  F_NL_SH = 16,                     // 8 bits: lane after O7
  F_LC_SH = 24                      // 2 bits: lc + 1
};

// ---- PTX helpers: mbarrier, bulk copy, named barrier --------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long *b, unsigned tx) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(b)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// profiling probes of earlier builds (no-ops)
#define KP_DECL
#define KP(idx, on) do {} while (0)
#define KPN(idx, on, n) do {} while (0)

// ---- small helpers -----------------------------------------------------------
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
__device__ __forceinline__ void put_inbox(InboxRec *dst, const InboxRec &rec) {
  int4 *d = reinterpret_cast<int4 *>(dst);
  const int4 *s = reinterpret_cast<const int4 *>(&rec);
  d[0] = s[0];
  d[1] = s[1];
}
__device__ __forceinline__ void red_add(long long *p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long *>(p), (unsigned long long)v);
}
__device__ __forceinline__ void record(const StepArgs &A, int vid, const Res &r, bool guard) {
  A.r_lc[vid] = (int8_t)r.lc;
  A.r_hand[vid] = (int8_t)(r.hand > 127 ? 127 : r.hand);
  A.r_acc[vid] = r.acc;
  A.r_fin[vid] = (int8_t)r.fin;
  A.r_guard[vid] = (uint8_t)(guard ? 1 : 0);
  A.r_mark[vid] = 1;
}

// Inboxes larger than a batch's pool (a tile taken alone, in global mode):
// rank / search through the record array in global memory.
__device__ __noinline__ void rank_inbox_global(const InboxRec *inb, int n_in, int *bsort, int t0,
                                               int nt) {
  for (int j = t0; j < n_in; j += nt) {
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

// Direct transport (NEXT-2): a mover entering another partition's
// tile is stored straight into the owner's inbox for t+1 and folded into the
// owner's summary / lane count with the same integer atomics a local mover
// uses, so no exchange or absorb step follows.  Returns 1 on inbox overflow.
__device__ __noinline__ int emit_peer(const StepArgs &A, const InboxRec &rec, int owner, int dt,
                                      int lane_g) {
  const PeerView &Q = A.peers[owner];
  const int nb = (step_t(A) + 1) & 1, ns = (step_t(A) + 1) % 3;
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

// A vehicle that leaves its slot: lane change / hand-off (kind 2) or arrival
// (kind 3).  Counters go to the tile's shared-memory accumulators.
__device__ __noinline__ void emit_moved(const StepArgs &A, const View &C, int i, const Res &r,
                                        int kind, TileSh &T) {
  const int vid = C.vid(i);
  if (r.lc != 0) atomicAdd(&T.c_lc, 1);
  if (r.hand) atomicAdd(&T.c_hand, r.hand);
  if (kind == 3) {
    A.status[vid] = ST_FINISHED;
    A.arrive_time[vid] = T.t + 1;
    A.wait_fin[vid] = r.wait1;
    atomicAdd(&T.c_fin, 1);
    long long *ta = A.tacc + (size_t)T.tile * kNAcc;
    const int ins = A.insert_time[vid];
    red_add(ta + ACC_SUM_TRAVEL, (long long)(T.t + 1 - ins));
    red_add(ta + ACC_SUM_INSERT, -(long long)ins);
    red_add(ta + ACC_SUM_WAIT_FIN, (long long)r.wait1);
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
  // the destination tile: this one (lane change, hand-off into its junction
  // lane), the exit lane's tile staged by k_prep, or the global tables
  int dt, dl, dib, dic, owner;
  if (r.cl >= 0) {
    dt = T.tile; dl = r.cl; dib = T.ibase; dic = T.icap; owner = A.rank;
  } else if (r.cx >= 0) {
    const ExtFirst &x = T.ext[r.cx - T.nroad];
    dt = x.dtile; dl = x.dlocal; dib = x.dibase; dic = x.dicap; owner = x.downer;
  } else {
    dt = A.lane_tile[r.lane_g]; dl = A.lane_local[r.lane_g];
    dib = A.tile_ibase[dt]; dic = A.tile_icap[dt]; owner = A.tile_owner[dt];
  }
  rec.meta = pack_meta(dl, m_prof(meta), r.cursor);
  rec.wait = r.wait1;
  rec.end_s = C.ends(i);
  if (owner == A.rank) {
    const int slot = atomicAdd(&A.icnt_out[dt], 1);
    if (slot < dic) put_inbox(A.vout + dib + slot, rec);
    else atomicAdd(&T.c_ovf, 1);
    atomicMin(&A.summ_next[r.lane_g], vkey(r.s1, vid));
    A.pubv_next[vid] = r.v1;
    if (A.lane_cnt_next) atomicAdd(&A.lane_cnt_next[r.lane_g], 1);
  } else if (A.peers) {                             // direct transport (NEXT-2)
    if (emit_peer(A, rec, owner, dt, r.lane_g)) atomicAdd(&T.c_ovf, 1);
  } else {                                          // migrant to another partition
    const int slot = atomicAdd(&A.out_cnt[owner], 1);
    if (slot < A.out_cap[owner]) {
      MigRec *m = A.out_buf + A.out_off[owner] + 1 + slot;
      put_inbox(&m->rec, rec);
      m->tile = dt;
      m->insert_time = A.insert_time[vid];
    } else {
      atomicAdd(&T.c_ovf, 1);
    }
  }
}

// ---- k_prep: what the step kernel reads from other tiles, staged per tile -----------------------
// One warp per own tile, one lane per tile lane (<= 32).  Junction lane: its
// signal at t and the first vehicle of its exit lane at t (the P:168-169
// lookahead target one lane beyond the tile: summary key, speed, length);
// road lane: the head of its pending-departure queue at t (K11).
// Written into the tile's block after its descriptor words, from where the
// step kernel bulk-copies them with the descriptor.  Also files the tile in
// the step kernel's work order.  Runs after k_signal (the signals of t) and
// reads only state(t).
__global__ void __launch_bounds__(128) k_prep(const __grid_constant__ StepArgs A) {
  pdl_wait();                                       // the signals of t (k_signal)
  pdl_trigger();
  const int w = blockIdx.x * 4 + (threadIdx.x >> 5), l = threadIdx.x & 31;
  if (w >= A.n_own) return;
  const int T = A.tiles[w];
  if (KW_ORDER && l == 0) {              // k_step_w's order: by vehicles at t, largest first
#if KW_ORDER == 2
    const int n = A.cnt_in[T] + A.icnt_in[T] + 4 * A.tinfo[3 * T + 1].z;   // + per-lane cost (DESIGN §5 fit)
#else
    const int n = A.cnt_in[T] + A.icnt_in[T];
#endif
    const int d = kNBucket - 1 - min(n >> KW_BSHIFT, kNBucket - 1);
    const int slot = atomicAdd(&A.bk_cnt[d], 1);
    A.bk_list[(size_t)d * A.n_tiles + slot] = T;
  }
  const int4 t1 = A.tinfo[3 * T + 1], t2 = A.tinfo[3 * T + 2];
  const int nl = t1.z, nroad = t1.w;
  int32_t *stage = A.desc + t1.x + t2.x;            // after the tile's descriptor words
  if (l >= nl) return;
  const int g = A.tile_lanes[A.tile_lane_off[T] + l];
  if (l >= nroad) {                                 // junction lane
    const int b = A.exit_lane[g];
    ExtFirst e;
    e.sig = A.lane_sig[g];
    e.b = b;
    e.Lb = A.lane_len[b];
    const int dt = A.lane_tile[b];
    e.dtile = dt;
    e.dlocal = A.lane_local[b];
    e.dibase = A.tile_ibase[dt];
    e.dicap = A.tile_icap[dt];
    e.downer = A.tile_owner[dt];
    unsigned long long key;
    const float *pv = A.pubv_cur;
    if (!A.peers) {
      key = A.summ_cur[b];
    } else {
      const int bt = A.lane_tile[b];
      if (A.tile_owner[bt] == A.rank) key = A.summ_cur[b];
      else key = peer_summary(A, bt, b, pv);
    }
    e.vid = -1;
    e.s = e.v = e.len = 0.f;
    if (key != kEmptyKey) {
      e.vid = (int)(unsigned)(key & 0xffffffffu);
      e.s = __uint_as_float((unsigned)(key >> 32));
      e.v = pv[e.vid];
      e.len = A.prof[A.veh_prof[e.vid]].len;
    }
    reinterpret_cast<ExtFirst *>(stage)[l - nroad] = e;
  } else {                                          // road lane
    PendHead ph;
    ph.k = -1;
    ph.depart = ph.prof = 0;
    ph.start_s = 0.f;
    ph.pad[0] = ph.pad[1] = ph.pad[2] = 0;
    const int h = A.pend_head[g];
    ph.h = h;
    if (h < A.pend_off[g + 1]) {
      const int vk = A.pend_vid[h];
      const int dep = A.depart[vk];
      if (dep <= step_t(A)) {
        ph.k = vk;
        ph.depart = dep;
        ph.start_s = A.start_s[vk];
        ph.prof = A.veh_prof[vk];
      }
    }
    reinterpret_cast<PendHead *>(stage + kExtWords * (nl - nroad))[l] = ph;
  }
}

// ---- per-lane order of the vehicles at t, as the step kernel merges them ---------------
// (a1): read side of sim_read_state.  One warp per own tile:
// the same merge as k_step's (stayers at own index + inbox keys below, inbox
// records at rank + stayers below, key (lane_local, s, vid)), written to
// vid[tile_base + position] / lane_local[tile_base + position].
__global__ void k_lane_order(const StepArgs A, int32_t *out_vid, uint8_t *out_lane) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= A.n_own) return;
  const int T = A.tiles[w];
  const int ns = A.cnt_in[T], ni = A.icnt_in[T], base = A.tile_base[T];
  const InboxRec *stay = tile_recs(A, T, ns);
  const InboxRec *inb = stay + ns;
  for (int i = lane; i < ns; i += 32) {
    const InboxRec x = stay[i];
    const unsigned long long h = hikey(m_lane(x.meta), x.s);
    int below = 0;
    for (int q = 0; q < ni; ++q) below += key_less(hikey(m_lane(inb[q].meta), inb[q].s), inb[q].vid, h, x.vid);
    out_vid[base + i + below] = x.vid;
    out_lane[base + i + below] = (uint8_t)m_lane(x.meta);
  }
  for (int r = lane; r < ni; r += 32) {
    const InboxRec x = inb[r];
    const unsigned long long h = hikey(m_lane(x.meta), x.s);
    int rank = 0;
    for (int q = 0; q < ni; ++q) rank += key_less(hikey(m_lane(inb[q].meta), inb[q].s), inb[q].vid, h, x.vid);
    int lo = 0, hi = ns;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const InboxRec &y = stay[mid];
      if (key_less(hikey(m_lane(y.meta), y.s), y.vid, h, x.vid)) lo = mid + 1; else hi = mid;
    }
    out_vid[base + rank + lo] = x.vid;
    out_lane[base + rank + lo] = (uint8_t)m_lane(x.meta);
  }
}
void launch_lane_order(const StepArgs &a, int32_t *out_vid, uint8_t *out_lane, void *stream) {
  if (a.n_own > 0) k_lane_order<<<(a.n_own + 7) / 8, 256, 0, (cudaStream_t)stream>>>(a, out_vid, out_lane);
}

void launch_prep(const StepArgs &a, void *stream) {
  if (a.n_own <= 0) return;
  launch_pdl(k_prep, dim3((a.n_own + 3) / 4), dim3(128), 0, (cudaStream_t)stream, a);
}

// ---- one tile ----------------------------------------------------
// Tile metadata from its descriptor into the warp's TileSh.
__device__ __forceinline__ void tile_setup(const Hdr &H, const int *W, const ExtFirst *ext,
                                           const PendHead *pend, const Prof *P, TileSh &T,
                                           int lane_id) {
  const int nl = H.nl, nroad = H.nroad;
  const int ne = W[2], n_all = W[3];
  const int eo = desc_ent_off(nl, nroad);
  const int to = eo + 8 * n_all;                     // target-road section
  if (lane_id == 0) {
    T.nl = nl;
    T.nroad = nroad;
    T.tile = H.tile;
    T.base = H.base;
    T.ibase = H.ibase;
    T.cap = H.cap;
    T.icap = H.icap;
    T.snap0 = 0;
    T.n = H.n_st + H.n_in;
    T.P = P;
    T.ext = ext;
    T.pend = pend;
    T.run = 0;
    T.c_fin = T.c_lc = T.c_hand = T.c_guard = T.c_ovf = T.c_ins = 0;
    T.c_delay = 0ull;
    T.ntr = W[to];
    T.umask = (uint32_t)W[to + 1];
    T.se_o = (uint32_t)(reinterpret_cast<const unsigned char *>(W + eo) - ks_smem);
    T.tr_o = (uint32_t)(reinterpret_cast<const unsigned char *>(W + to + 2) - ks_smem);
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
      int e0 = 0;                                    // entries of the road lanes before l
      for (int q = 0; q < l; ++q) e0 += (W[4 + 3 * nl + q] >> 8) & 0xff;
      T.se0[l] = (uint8_t)e0;
      const int *gw = W + 4 + 5 * nl + 6 * l;
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
  for (int ei = lane_id; ei < ne; ei += 32) {        // flags word -> SuccEnt::fl, in place
    int *ew = const_cast<int *>(W) + eo + 8 * ei;
    const unsigned fl = (unsigned)ew[3];
    const int jl = (int)(fl >> 24);
    const bool stop = (fl & 1u) && ext[jl - nroad].sig != SIG_GREEN;
    ew[3] = (stop ? 1 : 0) | ((int)(jl & 0xff) << 8);
  }
  __syncwarp();
}

// the vehicle at snapshot slot i has been updated (fp32 path or fp64
// canonical path): stayer results stay in the pass state for the in-order
// compaction, movers and arrivals leave now
template <class PS>
__device__ __forceinline__ void settle(const StepArgs &A, const PS &K, const View &C, int i,
                                       const Res &r, TileSh &T) {
  const int l = m_lane(C.meta(i));
  if (r.fin) {
    emit_moved(A, C, i, r, 3, T);
    K.kind(i) = 3;
  } else if (r.lc == 0 && r.hand == 0 && r.lane_g == T.glob[l]) {
    K.rs1(i) = r.s1;
    K.rv1(i) = r.v1;
    C.wait(i) = r.wait1;
    K.kind(i) = 1;
  } else {
    emit_moved(A, C, i, r, 2, T);
    K.kind(i) = 2;
  }
}

// pass 1: lane-change eligibility and O4-O6 on the current lane (fp32)
__device__ __forceinline__ void pass1(const StepArgs &A, const PState &K, const View &C, int i,
                                      const TileSh &T) {
  const uint32_t meta = C.meta(i);
  const int l = m_lane(meta);
  Me me;
  me.vid = C.vid(i);
  me.cur = m_cursor(meta);
  me.nxt = C.nxt(i);
  me.nxt2 = C.nxt2(i);
  me.ends = C.ends(i);
  const PV<float> p = pvals(T.P[m_prof(meta)], 0.f);
  const float s = C.s(i), v = C.v(i);
  const int lead = (i + 1 < T.seg_end[l]) ? i + 1 : -1;
  if (A.record) {
    const int of = (i > T.seg_start[l]) ? i - 1 : -1;
    A.r_of[me.vid] = of >= 0 ? C.vid(of) : -1;
    for (int q = 0; q < 4; ++q) A.r_side[4 * me.vid + q] = -1;
  }
  Guard g;
  g.hit = false;
  Elig E;
  E.sl0 = E.sl1 = -1;
  E.mand = 0;
  E.inG = true;
  E.want0 = E.want1 = false;
  me.k = -1;
  if (T.isroad[l]) E = lc_elig<float, kGuard>(A, T, l, s, v, p, me, g);
  const LEv<float> use = eval_lane<float, kGuard>(A, T, C, l, lead, s, v, p, me, g);
  if (A.record) {
    A.r_leader[me.vid] = use.leader;
    A.r_hops[me.vid] = (int8_t)use.hops;
    A.r_phantom[me.vid] = (int8_t)use.phantom;
  }
  K.pa(i) = use.a;
  K.plim(i) = use.lim;
  K.plimrel(i) = use.limrel;
  K.pvlim(i) = use.vlim;
  K.pnext1(i) = use.next1;
  K.pnl(i) = (uint8_t)(use.nl1 < 0 ? 0xff : use.nl1);
  K.pfl(i) = (use.has_lim ? F_LIM : 0u) | (g.hit ? F_HIT : 0u) | (E.inG ? F_ING : 0u) |
             (E.want0 ? F_W0 : 0u) | (E.want1 ? F_W1 : 0u) | ((uint32_t)(E.mand + 1) << F_MAND_SH) |
             ((uint32_t)(me.k + 1) << F_K_SH) | ((uint32_t)l << F_NL_SH) | (1u << F_LC_SH);
}

// pass 2: O7 (MOBIL) for a vehicle that may change lane (fp32)
__device__ __forceinline__ void pass2(const StepArgs &A, const PState &K, const View &C, int i,
                                      const TileSh &T) {
  const uint32_t meta = C.meta(i);
  const int l = m_lane(meta);
  const uint32_t fl = K.pfl(i);
  Me me;
  me.vid = C.vid(i);
  me.cur = m_cursor(meta);
  me.nxt = C.nxt(i);
  me.nxt2 = C.nxt2(i);
  me.ends = C.ends(i);
  me.k = (int)((fl >> F_K_SH) & 31u) - 1;
  const PV<float> p = pvals(T.P[m_prof(meta)], 0.f);
  const float s = C.s(i), v = C.v(i);
  Elig E;
  E.sl0 = T.left[l];
  E.sl1 = T.right[l];
  E.mand = (int)((fl >> F_MAND_SH) & 3u) - 1;
  E.inG = (fl & F_ING) != 0;
  E.want0 = (fl & F_W0) != 0;
  E.want1 = (fl & F_W1) != 0;
  Guard g;
  g.hit = false;
  const SideRes<float> sr = lc_decide<float, kGuard>(A, T, C, i, l, s, v, p, me, E, K.pa(i), g);
  if (g.hit) {
    K.pfl(i) = fl | F_HIT;
  } else if (sr.choice >= 0) {
    K.pa(i) = sr.a;
    K.plim(i) = sr.lim;
    K.plimrel(i) = sr.limrel;
    K.pvlim(i) = sr.vlim;
    K.pnext1(i) = sr.next1;
    K.pnl(i) = (uint8_t)(sr.nl1 < 0 ? 0xff : sr.nl1);
    const int nl = sr.choice == 0 ? E.sl0 : E.sl1;
    const int lc = sr.choice == 0 ? -1 : 1;
    K.pfl(i) = (fl & ~(F_LIM | (0xffu << F_NL_SH) | (3u << F_LC_SH))) | (sr.has_lim ? F_LIM : 0u) |
               ((uint32_t)nl << F_NL_SH) | ((uint32_t)(lc + 1) << F_LC_SH);
  }
}

// pass 3: O8-O9 (fp32).  Returns false if the vehicle must be recomputed.
__device__ __forceinline__ bool pass3(const StepArgs &A, const PState &K, const View &C, int i,
                                      TileSh &T) {
  const uint32_t fl = K.pfl(i);
  if (fl & F_HIT) return false;
  const uint32_t meta = C.meta(i);
  Me me;
  me.vid = C.vid(i);
  me.cur = m_cursor(meta);
  me.nxt = C.nxt(i);
  me.nxt2 = C.nxt2(i);
  me.ends = C.ends(i);
  me.k = -1;
  LEv<float> use;
  use.a = K.pa(i);
  use.lim = K.plim(i);
  use.limrel = K.plimrel(i);
  use.vlim = K.pvlim(i);
  use.next1 = K.pnext1(i);
  use.nl1 = K.pnl(i) == 0xff ? -1 : (int)K.pnl(i);
  use.has_lim = (fl & F_LIM) != 0;
  const int new_l = (int)((fl >> F_NL_SH) & 0xffu);
  const int lc = (int)((fl >> F_LC_SH) & 3u) - 1;
  Guard g;
  g.hit = false;
  Res r;
  integrate<float, kGuard>(A, T, C.s(i), C.v(i), me, use, lc, new_l, C.wait(i), r, g);
  if (g.hit) return false;
  if (A.record) record(A, me.vid, r, false);
  settle(A, K, C, i, r, T);
  return true;
}

// the fp64 canonical recomputation of one vehicle
template <class PS>
__device__ __noinline__ void pass_fp64(const StepArgs &A, const PS &K, const View &C, int i,
                                       TileSh &T) {
  Res r;
  Guard g;
  g.hit = false;
  veh_update<double, false>(A, T, C, i, r, g);
  if (A.record) record(A, C.vid(i), r, true);
  settle(A, K, C, i, r, T);
}

// warp-aggregated append to a per-tile list
__device__ __forceinline__ int push_list(bool pred, uint16_t *list, int count, int val, int lane) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (pred) list[count + __popc(m & ((1u << lane) - 1u))] = (uint16_t)val;
  return count + __popc(m);
}

// passes 1-3 and the fp64 recomputation over the tile's n snapshot slots
template <bool EXACT>
__device__ __forceinline__ void run_passes(const StepArgs &A, const PState &K, const View &C,
                                           TileSh &T, int n, int lane) {
  KP_DECL
  int nd = 0;
  if constexpr (!EXACT) {
    int nc = 0;
    for (int q0 = 0; q0 < n; q0 += 32) {             // pass 1 (every vehicle)
      const int q = q0 + lane;
      bool cand = false;
      if (q < n) {
        pass1(A, K, C, q, T);
        const uint32_t fl = K.pfl(q);
        cand = !(fl & F_HIT) && ((fl & (F_W0 | F_W1)) || (A.record && T.isroad[m_lane(C.meta(q))]));
      }
      nc = push_list(cand, K.cand(), nc, q, lane);
    }
    __syncwarp();
    KP(25, lane == 0);
    for (int q = lane; q < nc; q += 32) pass2(A, K, C, K.cand()[q], T);   // pass 2 (compacted)
    __syncwarp();
    KP(26, lane == 0);
    for (int q0 = 0; q0 < n; q0 += 32) {             // pass 3 (every vehicle)
      const int q = q0 + lane;
      bool def = false;
      if (q < n) def = !pass3(A, K, C, q, T);
      nd = push_list(def, K.defl(), nd, q, lane);
    }
    __syncwarp();
    KP(27, lane == 0);
  } else {
    for (int q = lane; q < n; q += 32) K.defl()[q] = (uint16_t)q;
    nd = n;
    __syncwarp();
  }
  for (int q = lane; q < nd; q += 32) {              // fp64 canonical path
    pass_fp64(A, K, C, K.defl()[q], T);
    if (!EXACT) atomicAdd(&T.c_guard, 1);
  }
  __syncwarp();
  KP(28, lane == 0);
}

// In-order compaction of the tile's stayers into its record region for t+1,
// right-aligned (so that they and the inbox the tile receives form one
// contiguous range): the stayer count first, then each stayer
// to base + cap - count + rank as one 32-B record (coalesced); the first
// stayer of each lane is remembered for the t+1 summary.
template <class PS>
__device__ __forceinline__ void compact(const StepArgs &A, const PS &K, const View &C, TileSh &T,
                                        int n, int lane_id) {
  int cnt = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane_id;
    cnt += __popc(__ballot_sync(0xffffffffu, i < n && K.kind(i) == 1));
  }
  if (cnt > T.cap) {                                // slab capacity exceeded: sticky SIM_E_CAPACITY
    if (lane_id == 0) atomicAdd(&T.c_ovf, cnt - T.cap);
    cnt = T.cap;
  }
  InboxRec *dst = A.vout + T.base + T.cap - cnt;
  int run = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane_id;
    const bool st = i < n && K.kind(i) == 1;
    const unsigned ball = __ballot_sync(0xffffffffu, st);
    if (st) {
      const int rank = run + __popc(ball & ((1u << lane_id) - 1u));
      if (rank < cnt) {
        const uint32_t meta = C.meta(i);
        InboxRec r;
        r.s = K.rs1(i);
        r.v = K.rv1(i);
        r.vid = C.vid(i);
        r.nxt = C.nxt(i);
        r.nxt2 = C.nxt2(i);
        r.meta = meta;
        r.wait = C.wait(i);
        r.end_s = C.ends(i);
        put_inbox(dst + rank, r);
        atomicMin(&T.first_out[m_lane(meta)], (rank << 15) | i);
      }
    }
    run += __popc(ball);
  }
  __syncwarp();
  if (lane_id == 0) T.run = cnt;
  __syncwarp();
}

// departure onto road lane l of the tile (K11; ledger L25): the head of
// its pending queue, if due, is inserted when the gaps to the vehicles ahead
// and behind its start position allow it (against state(t)).  Out of line.
__device__ __noinline__ void depart(const StepArgs &A, const View &C, TileSh &T, int l) {
  const int tile = T.tile;
  const PendHead ph = T.pend[l];
  const int g = T.glob[l];
  const int k = ph.k;
  const double ss = (double)ph.start_s;
  const Prof &pk = T.P[ph.prof];
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
  if (!ok) return;
  InboxRec rec;
  rec.s = (float)ss;
  rec.v = 0.f;
  rec.vid = k;
  const int off = A.route_start[k], rl = A.route_len[k];
  rec.nxt = rl > 1 ? A.route[off + 1] : -1;
  rec.nxt2 = rl > 2 ? A.route[off + 2] : -1;
  rec.meta = pack_meta(l, ph.prof, 0);
  rec.wait = 0;
  rec.end_s = A.end_s[k];
  const int slot = atomicAdd(&A.icnt_out[tile], 1);
  if (slot < T.icap) put_inbox(A.vout + T.ibase + slot, rec);
  else atomicAdd(&T.c_ovf, 1);
  atomicMin(&A.summ_next[g], vkey(rec.s, k));
  A.pubv_next[k] = 0.f;
  if (A.lane_cnt_next) atomicAdd(&A.lane_cnt_next[g], 1);
  A.pend_head[g] = ph.h + 1;
  A.status[k] = ST_DRIVING;
  A.insert_time[k] = T.t + 1;
  if (A.record) A.r_ins[k] = 1;
  atomicAdd(&T.c_ins, 1);
  atomicAdd(&T.c_delay, (unsigned long long)(long long)(T.t + 1 - ph.depart));
}

// Lane summaries for t+1, departures (K11; L25) and counters (a6) of
// the tile, after all its vehicles are settled.
template <class PS>
__device__ __forceinline__ void tile_finish(const StepArgs &A, const PS &K, const View &C,
                                            TileSh &T, int lane_id) {
  const int nl = T.nl, nroad = T.nroad, tile = T.tile;
  const int run = T.run < T.cap ? T.run : T.cap;
  for (int l = lane_id; l < nl; l += 32) {
    const int g = T.glob[l];
    const int fo = T.first_out[l];
    if (fo != 0x7fffffff) {
      const int rank = fo >> 15, idx = fo & 0x7fff;
      const int vid = C.vid(idx);
      atomicMin(&A.summ_next[g], vkey(K.rs1(idx), vid));
      A.pubv_next[vid] = K.rv1(idx);
      if (A.lane_cnt_next) {                          // stayers of lane l: [rank, next lane's first)
        int end = run;
        for (int q = l + 1; q < nl; ++q)
          if (T.first_out[q] != 0x7fffffff) { end = T.first_out[q] >> 15; break; }
        atomicAdd(&A.lane_cnt_next[g], end - rank);
      }
    }
    A.summ_clear[g] = kEmptyKey;
  }
  if (lane_id < nroad && T.pend[lane_id].k >= 0 && T.usable[lane_id]) depart(A, C, T, lane_id);
  __syncwarp();
  if (lane_id == 0) {
    long long *ta = A.tacc + (size_t)tile * kNAcc;
    red_add(ta + ACC_VEH_STEPS, T.n);
    if (T.c_fin) red_add(ta + ACC_FINISHED, T.c_fin);
    if (T.c_ins) {
      red_add(ta + ACC_INSERTED, T.c_ins);
      red_add(ta + ACC_SUM_DELAY, (long long)T.c_delay);
      red_add(ta + ACC_SUM_INSERT, (long long)T.c_ins * (T.t + 1));   // insert_time = t + 1
    }
    if (T.c_lc) red_add(ta + ACC_LANE_CHANGES, T.c_lc);
    if (T.c_hand) red_add(ta + ACC_HANDOFFS, T.c_hand);
    if (T.c_guard) red_add(ta + ACC_GUARD, T.c_guard);
    if (T.c_ovf) red_add(ta + ACC_OVERFLOW, T.c_ovf);
    A.cnt_out[tile] = run;
    A.icnt_in[tile] = 0;
  }
  __syncwarp();
}

// one tile, start to finish, by one consumer warp
// GM: the tile is in global mode.  A separate instantiation, so that in the
// common one every snapshot / pass-state access is provably to shared memory
// (LDS/STS instead of generic loads).
template <bool EXACT, bool GM>
__device__ __forceinline__ void run_tile(const StepArgs &A, unsigned char *slot, const Hdr &H, TileSh &T,
                                         const Prof *P, int lane) {
  KP_DECL
  const int ns = H.n_st, ni = H.n_in, n = ns + ni;
  const SlotLayout L = GM ? slot_layout(0, 0, H.dw) : slot_layout(ns, ni, H.dw);
  const int *W = reinterpret_cast<const int *>(slot + L.desc);
  if (lane == 0) T.t = step_t(A);                   // tile_setup ends with __syncwarp
  tile_setup(H, W, reinterpret_cast<const ExtFirst *>(W + H.dwd),
             reinterpret_cast<const PendHead *>(W + H.dwd + kExtWords * (H.nl - H.nroad)), P, T, lane);
  KP(22, lane == 0);
  View C;
  PState K;
  if (!GM) {
    C.p = reinterpret_cast<uint32_t *>(slot + L.snap);
    C.st = L.n4;
    K = pstate_at(slot + L.veh, L.n4);                // after the merge (below)
  } else {
    const size_t o = (size_t)H.base;
    C.st = H.cap + H.icap;
    C.p = A.scratch + 8 * o;
    const size_t o2 = o + 4 * (size_t)H.tile;       // 4 slots of slack per tile: 16-B strides
    K = pstate_at(reinterpret_cast<unsigned char *>(A.pscratch + 10 * o2), (C.st + 3) & ~3);
  }
  auto put = [&](int pos, const InboxRec &x) {
    C.s(pos) = x.s;
    C.v(pos) = x.v;
    C.vid(pos) = x.vid;
    C.meta(pos) = x.meta;
    C.nxt(pos) = x.nxt;
    C.nxt2(pos) = x.nxt2;
    C.wait(pos) = x.wait;
    C.ends(pos) = x.end_s;
  };
  // ---- merge stayers + sorted inbox into the snapshot (a1) --------------------------
  // stayers (in order, L23 keeps them so) at own index + #inbox keys below;
  // inbox records at their rank + #stayers below: O(n + m log n), no sort
  if (!GM) {
    const InboxRec *stay = reinterpret_cast<const InboxRec *>(slot + L.veh);
    const InboxRec *inb = stay + ns;
    unsigned long long *skh = reinterpret_cast<unsigned long long *>(slot + L.sortk);
    int *skv = reinterpret_cast<int *>(skh + ni);
    int *bs = skv + ni;
    for (int r = lane; r < ni; r += 32) {            // inbox keys ranked
      const InboxRec &x = inb[r];
      const unsigned long long h = hikey(m_lane(x.meta), x.s);
      int rank = 0;
      for (int q = 0; q < ni; ++q) {
        const InboxRec &o = inb[q];
        rank += key_less(hikey(m_lane(o.meta), o.s), o.vid, h, x.vid);
      }
      skh[rank] = h;
      skv[rank] = x.vid;
      bs[rank] = r;
    }
    __syncwarp();
    for (int i = lane; i < ns; i += 32) {
      const InboxRec x = stay[i];
      int lo = 0, hi = ni;
      if (ni > 0) {
        const unsigned long long h = hikey(m_lane(x.meta), x.s);
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (key_less(skh[mid], skv[mid], h, x.vid)) lo = mid + 1; else hi = mid;
        }
      }
      put(i + lo, x);
    }
    for (int r = lane; r < ni; r += 32) {
      const InboxRec x = inb[bs[r]];
      const unsigned long long h = skh[r];
      int lo = 0, hi = ns;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const InboxRec &y = stay[mid];
        if (key_less(hikey(m_lane(y.meta), y.s), y.vid, h, x.vid)) lo = mid + 1; else hi = mid;
      }
      put(r + lo, x);
    }
  } else {
    const InboxRec *stay = tile_recs(A, H.tile, ns);
    const InboxRec *inb = stay + ns;
    const int *bsort = A.bsort_scratch + H.ibase;
    if (ni > 0) rank_inbox_global(inb, ni, A.bsort_scratch + H.ibase, lane, 32);
    __syncwarp();
    for (int i = lane; i < ns; i += 32) {
      const InboxRec x = stay[i];
      const int lo = ni > 0 ? lower_bound_inbox_global(inb, bsort, ni, hikey(m_lane(x.meta), x.s), x.vid) : 0;
      put(i + lo, x);
    }
    for (int r = lane; r < ni; r += 32) {
      const InboxRec x = inb[bsort[r]];
      const unsigned long long h = hikey(m_lane(x.meta), x.s);
      int lo = 0, hi = ns;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const InboxRec &y = stay[mid];
        if (key_less(hikey(m_lane(y.meta), y.s), y.vid, h, x.vid)) lo = mid + 1; else hi = mid;
      }
      put(r + lo, x);
    }
  }
  __syncwarp();
  KP(23, lane == 0);
  // ---- lane segments of the snapshot -------------------------------------------------
  for (int i = lane; i < n; i += 32) {
    const int l = m_lane(C.meta(i));
    if (i == 0 || m_lane(C.meta(i - 1)) != l) T.seg_start[l] = (int16_t)i;
    if (i == n - 1 || m_lane(C.meta(i + 1)) != l) T.seg_end[l] = (int16_t)(i + 1);
  }
  __syncwarp();
  KP(24, lane == 0);
  run_passes<EXACT>(A, K, C, T, n, lane);
  compact(A, K, C, T, n, lane);
  KP(29, lane == 0);
  tile_finish(A, K, C, T, lane);
  KP(30, lane == 0);
}

// global-mode tiles (rare), out of line so their copy of the passes stays out
// of the hot code
template <bool EXACT>
__device__ __noinline__ void run_tile_gm(const StepArgs &A, unsigned char *slot, const Hdr &H, TileSh &T,
                                         const Prof *P, int lane) {
  run_tile<EXACT, true>(A, slot, H, T, P, lane);
}

// ---- the step kernel k_step_w ---------------------
// The round-1 execution model on this round's data layout and model code: one
// warp per CTA, many CTAs per SM, no producer, no rounds.  Each warp claims a
// tile, bulk-copies its block (descriptor + k_prep staging) into its own
// shared area, merges the tile's records from global memory into a shared
// snapshot, runs the fused per-vehicle update (veh_update: O4-O9 in one pass)
// and the fp64 recomputation of guard hits, compacts and finishes the tile.
// Tiles whose snapshot does not fit the area run in global mode.
#ifndef KW_BLOCKS
#define KW_BLOCKS 16
#endif
#ifndef KW_MINB
#define KW_MINB KW_BLOCKS                            // launch-bounds CTAs per SM (register cap)
#endif
constexpr int kWB = KW_BLOCKS;                       // one-warp CTAs per SM
// pass state of the fused path: the stayer results and the fp64 list only
struct PStateM {
  unsigned char *p;
  int n4;
  __device__ __forceinline__ float &rs1(int i) const { return reinterpret_cast<float *>(p)[i]; }
  __device__ __forceinline__ float &rv1(int i) const { return reinterpret_cast<float *>(p)[n4 + i]; }
  __device__ __forceinline__ uint8_t &kind(int i) const { return p[8 * n4 + i]; }
  __device__ __forceinline__ uint16_t *defl() const { return reinterpret_cast<uint16_t *>(p + 9 * n4); }
};
struct WHead {
  unsigned long long bar;                           // the block copy's mbarrier
  Hdr H;
  TileSh T;
};
constexpr int kWBlockSmem = (228 * 1024) / kWB - 1024;   // per CTA (1 KB reserved per CTA)
constexpr int kWHead = ((int)sizeof(WHead) + 127) & ~127;
constexpr int kWArea = (kWBlockSmem - kWHead) & ~127;
struct __align__(128) WSmem {
  WHead h;
  __align__(128) unsigned char area[kWArea];
};
static_assert(sizeof(WSmem) <= kWBlockSmem, "WSmem fits the per-CTA budget");

template <bool EXACT>
__device__ __forceinline__ void wtile(const StepArgs &A, WSmem &M, int tile, unsigned &phase,
                                      int lane) {
  TileSh &T = M.h.T;
  Hdr &H = M.h.H;
  const int4 t0 = A.tinfo[3 * tile], t1 = A.tinfo[3 * tile + 1], t2 = A.tinfo[3 * tile + 2];
  const int ns = A.cnt_in[tile], ni = A.icnt_in[tile], n = ns + ni;
  const int dw = t1.y;
  const int n4 = (n + 3) & ~3;
  // area: block (4 dw B) | snapshot (32 n4 B) | pass state (11 n4 B, 16-B rounded) | inbox keys (16 ni B)
  const uint32_t o_snap = 4u * (uint32_t)dw;
  const uint32_t o_pass = o_snap + 32u * (uint32_t)n4;
  const uint32_t o_sk = o_pass + ((11u * (uint32_t)n4 + 15u) & ~15u);
  const bool gm = o_sk + 16u * (uint32_t)ni > (uint32_t)kWArea;
  if (lane == 0) {
    H.tile = tile; H.n_st = ns; H.n_in = ni; H.base = t0.x; H.ibase = t0.y; H.cap = t0.z;
    H.icap = t0.w; H.nl = t1.z; H.nroad = t1.w; H.dw = dw; H.dwd = t2.x; H.gm = gm ? 1 : 0;
    H.done = 0; H.off = 0;
    fence_proxy_async();                            // the area's generic writes of the last tile
    mbar_arrive_tx(&M.h.bar, 4u * (unsigned)dw);
    bulk_g2s(M.area, A.desc + t1.x, 4u * (unsigned)dw, &M.h.bar);
  }
  mbar_wait(&M.h.bar, phase);
  phase ^= 1u;
  __syncwarp();
  if (gm) {                                         // block at offset 0 = slot_layout(0, 0, dw).desc
    run_tile_gm<EXACT>(A, M.area, H, T, A.prof, lane);
    return;
  }
  const int *W = reinterpret_cast<const int *>(M.area);
  if (lane == 0) T.t = step_t(A);
  tile_setup(H, W, reinterpret_cast<const ExtFirst *>(W + H.dwd),
             reinterpret_cast<const PendHead *>(W + H.dwd + kExtWords * (H.nl - H.nroad)), A.prof, T,
             lane);
  View C;
  C.p = reinterpret_cast<uint32_t *>(M.area + o_snap);
  C.st = n4;
  PStateM K;
  K.p = M.area + o_pass;
  K.n4 = n4;
  auto put = [&](int pos, const InboxRec &x) {
    C.s(pos) = x.s;
    C.v(pos) = x.v;
    C.vid(pos) = x.vid;
    C.meta(pos) = x.meta;
    C.nxt(pos) = x.nxt;
    C.nxt2(pos) = x.nxt2;
    C.wait(pos) = x.wait;
    C.ends(pos) = x.end_s;
  };
  // merge (a1) from the records in global memory: inbox keys ranked into
  // shared memory, stayers at own index + #inbox keys below, inbox records at
  // rank + #stayers below
  const InboxRec *stay = tile_recs(A, tile, ns);
  const InboxRec *inb = stay + ns;
  unsigned long long *skh = reinterpret_cast<unsigned long long *>(M.area + o_sk);
  int *skv = reinterpret_cast<int *>(skh + ni);
  int *bs = skv + ni;
  for (int r = lane; r < ni; r += 32) {
    const InboxRec x = inb[r];
    const unsigned long long h = hikey(m_lane(x.meta), x.s);
    int rank = 0;
    for (int q = 0; q < ni; ++q) {
      const InboxRec o = inb[q];
      rank += key_less(hikey(m_lane(o.meta), o.s), o.vid, h, x.vid);
    }
    skh[rank] = h;
    skv[rank] = x.vid;
    bs[rank] = r;
  }
  __syncwarp();
  for (int i = lane; i < ns; i += 32) {
    const InboxRec x = stay[i];
    int lo = 0, hi = ni;
    if (ni > 0) {
      const unsigned long long h = hikey(m_lane(x.meta), x.s);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key_less(skh[mid], skv[mid], h, x.vid)) lo = mid + 1; else hi = mid;
      }
    }
    put(i + lo, x);
  }
  for (int r = lane; r < ni; r += 32) {
    const InboxRec x = inb[bs[r]];
    const unsigned long long h = skh[r];
    int lo = 0, hi = ns;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const InboxRec &y = stay[mid];
      if (key_less(hikey(m_lane(y.meta), y.s), y.vid, h, x.vid)) lo = mid + 1; else hi = mid;
    }
    put(r + lo, x);
  }
  __syncwarp();
  for (int i = lane; i < n; i += 32) {              // lane segments of the snapshot
    const int l = m_lane(C.meta(i));
    if (i == 0 || m_lane(C.meta(i - 1)) != l) T.seg_start[l] = (int16_t)i;
    if (i == n - 1 || m_lane(C.meta(i + 1)) != l) T.seg_end[l] = (int16_t)(i + 1);
  }
  __syncwarp();
  // the fused per-vehicle update; guard hits and exact mode go to the fp64 path
  int nd = 0;
  if constexpr (!EXACT) {
    for (int q0 = 0; q0 < n; q0 += 32) {
      const int q = q0 + lane;
      bool def = false;
      if (q < n) {
        Res r;
        Guard g;
        g.hit = false;
        veh_update<float, kGuard>(A, T, C, q, r, g);
        if (g.hit) {
          def = true;
        } else {
          if (A.record) record(A, C.vid(q), r, false);
          settle(A, K, C, q, r, T);
        }
      }
      nd = push_list(def, K.defl(), nd, q, lane);
    }
  } else {
    for (int q = lane; q < n; q += 32) K.defl()[q] = (uint16_t)q;
    nd = n;
  }
  __syncwarp();
  for (int q = lane; q < nd; q += 32) {
    pass_fp64(A, K, C, K.defl()[q], T);
    if (!EXACT) atomicAdd(&T.c_guard, 1);
  }
  __syncwarp();
  compact(A, K, C, T, n, lane);
  tile_finish(A, K, C, T, lane);
}

#ifdef KW_TAIL
__device__ unsigned long long g_kw_fin[4096];
#endif
template <bool EXACT>
__global__ void __launch_bounds__(32, KW_MINB) k_step_w(const __grid_constant__ StepArgs A) {
  WSmem &M = *reinterpret_cast<WSmem *>(ks_smem);
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(&M.h.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  pdl_wait();
  pdl_trigger();
  unsigned phase = 0;
  // this step's tile order (KW_ORDER): exclusive prefix of the bucket counts,
  // buckets lane and 32 + lane in this lane
  int e0 = 0, e1 = 0;
  if (KW_ORDER) {
    static_assert(kNBucket == 64, "two buckets per lane");
    const int c0 = A.bk_cnt[lane], c1 = A.bk_cnt[32 + lane];
    int i0 = c0, i1 = c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(0xffffffffu, i0, o), y1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) { i0 += y0; i1 += y1; }
    }
    const int t0 = __shfl_sync(0xffffffffu, i0, 31);
    e0 = i0 - c0;
    e1 = t0 + i1 - c1;
  }
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&A.work[0], 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= A.n_own) break;
    int tile;
    if (KW_ORDER) {                                 // the last bucket d with prefix[d] <= c
      const unsigned m0 = __ballot_sync(0xffffffffu, e0 <= c), m1 = __ballot_sync(0xffffffffu, e1 <= c);
      const int d = m1 ? 32 + (31 - __clz(m1)) : 31 - __clz(m0);
      const int pre = __shfl_sync(0xffffffffu, d >= 32 ? e1 : e0, d & 31);
      tile = A.bk_list[(size_t)d * A.n_tiles + (c - pre)];
    } else {
      tile = A.tiles[c];
    }
    wtile<EXACT>(A, M, tile, phase, lane);
    __syncwarp();
  }
#ifdef KW_TAIL
  if (lane == 0 && blockIdx.x < 4096) {             // dev builds: per-CTA finish time
    unsigned long long tnow;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
    g_kw_fin[blockIdx.x] = tnow;
  }
#endif
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(&A.work[1], 1) == (int)gridDim.x - 1) {
      A.work[0] = 0;
      A.work[1] = 0;
      if (KW_ORDER)
        for (int d = 0; d < kNBucket; ++d) A.bk_cnt[d] = 0;   // for the next step's k_prep
    }
  }
}

int step_smem_bytes() { return (int)sizeof(WSmem); }

}  // namespace sim

// dev builds (-DKW_TAIL): per-CTA finish times of the last k_step_w
extern "C" int sim_debug_kw_finish(unsigned long long *out) {
#ifdef KW_TAIL
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, sim::g_kw_fin, sizeof(sim::g_kw_fin));
  return 4096;
#else
  (void)out;
  return 0;
#endif
}

namespace sim {

static int resident[2] = {0, 0};                    // resident CTAs per GPU, per instantiation
void init_step_launch(int smem_bytes) {
  if (!resident[0]) {
    int dev = 0, nsm = 0, b0 = 0, b1 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_step_w<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_step_w<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, k_step_w<false>, 32, smem_bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_step_w<true>, 32, smem_bytes);
    resident[0] = std::max(1, b0) * std::max(1, nsm);
    resident[1] = std::max(1, b1) * std::max(1, nsm);
  }
}

void launch_step(const StepArgs &a, void *stream, int smem_bytes) {
  init_step_launch(smem_bytes);
  if (a.n_own <= 0) return;
  const int ex = a.exact_mode ? 1 : 0;
  const int grid = std::min(a.n_own, resident[ex]);  // one warp per CTA, persistent
  if (ex) launch_pdl(k_step_w<true>, dim3(grid), dim3(32), smem_bytes, (cudaStream_t)stream, a);
  else launch_pdl(k_step_w<false>, dim3(grid), dim3(32), smem_bytes, (cudaStream_t)stream, a);
}

}  // namespace sim
