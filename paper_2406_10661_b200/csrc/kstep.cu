// kstep.cu — the fused step kernel k_step (rows a0-a4, a6).
//
// A warp-specialised persistent kernel.  Each CTA has one PRODUCER warp and
// kCW CONSUMER warps and works through BATCHES of road tiles (a tile = one
// road's lanes + the junction lanes leaving it, dev.h):
//
//   producer  claims tiles from a global work counter (largest first), packs
//             consecutive ones into a batch of at most kBatch vehicles, and
//             streams the batch's stayer slab segments, inbox records and
//             tile descriptors into a shared-memory stage with 1-D bulk copies
//             (cp.async.bulk + mbarrier complete_tx).  It also gathers what
//             the batch needs from other tiles — the first vehicle of every
//             junction lane's exit lane at t (the P:168-169 lookahead target),
//             the junction lanes' signals, the heads of the pending-departure
//             queues — so the consumers' critical path has no global loads in
//             the common case.  kStages stages form a ring (full / empty
//             mbarriers), so batch b+1 streams in while batch b is computed.
//   consumers run the batch in dense phases separated by a named barrier:
//             tile metadata; merge of in-order stayers + sorted inbox into
//             the snapshot (a1); pass 1 = eligibility +
//             leader / lookahead + IDM on the current lane for every vehicle
//             (a2, a3); pass 2 = MOBIL for the compacted list of vehicles that
//             may change lane; pass 3 = integrate / hand-off /
//             arrival (a4) with movers emitted to their destination inbox;
//             the fp64 canonical recomputation of vehicles whose fp32 margins
//             fell inside the guard band; then per tile the
//             in-order compaction of stayers, lane summaries for t+1,
//             departures (K11) and counters (a6).
//
// Every decision reads only state(t) (the snapshot) and all
// cross-tile outputs are integer atomics into the t+1 buffers, so the result
// does not depend on which CTA takes which tile or in what order.
#include <cuda_runtime.h>

#include <algorithm>

#include "dev.h"
#include "model.cuh"

namespace sim {

#ifndef KS_CONS_WARPS
#define KS_CONS_WARPS 8
#endif
#ifndef KS_BATCH
#define KS_BATCH 352
#endif
#ifndef KS_MAXT
#define KS_MAXT 10
#endif
#ifndef KS_STAGES
#define KS_STAGES 2
#endif
constexpr int kCW = KS_CONS_WARPS;            // consumer warps
constexpr int kCT = kCW * 32;                 // consumer threads
constexpr int kStepThreads = kCT + 32;        // + the producer warp (the last warp)
constexpr int kBatch = KS_BATCH;              // vehicle slots of a batch
constexpr int kMaxT = KS_MAXT;                // tiles per batch
constexpr int kStages = KS_STAGES;
constexpr int kInPool = 160;                  // inbox records per batch
constexpr int kDescPool = 1280;               // descriptor words per batch
constexpr int kXPool = 80;                    // junction lanes per batch (gathered exit-lane firsts)
constexpr int kPPool = 40;                    // road lanes per batch (pending-queue heads)
constexpr int kSlabWords = 7 * kBatch + 7 * 3 * kMaxT;   // stayer fields, each padded to 4 elements
constexpr int kGroup = 16;                    // tiles claimed from the work counter at a time
constexpr int kCBar = 1;                      // named barrier of the consumer warps
static_assert(kBatch % 32 == 0 && kBatch < 32768, "batch slots");
static_assert(kGroup * 2 <= 32, "the producer warp holds two groups");

struct BatchHdr {
  int nt, gmode, done, nveh, nst, nin;
  int tile[kMaxT], n_st[kMaxT], n_in[kMaxT], base[kMaxT], ibase[kMaxT], cap[kMaxT], icap[kMaxT];
  int nl[kMaxT], nroad[kMaxT], doff[kMaxT], dw[kMaxT];
  int slab[kMaxT], r4[kMaxT];       // stage word offset of the tile's 7 stayer arrays, their stride
  int in0[kMaxT];                   // flat inbox offset (stage record offset)
  int st0[kMaxT];                   // flat stayer offset
  int desc[kMaxT];                  // stage word offset of the descriptor
  int xo[kMaxT], po[kMaxT];         // gather offsets (junction lanes, road lanes)
  int snap0[kMaxT];                 // flat snapshot offset
};

struct __align__(16) Stage {
  unsigned long long full, empty;   // mbarriers
  BatchHdr H;
  __align__(16) uint32_t slab[kSlabWords];
  InboxRec inbox[kInPool];
  __align__(16) int32_t desc[kDescPool];
  ExtFirst ext[kXPool];
  PendHead pend[kPPool];
};

struct __align__(16) Cons {
  uint32_t snap[7 * kBatch];        // snapshot of the batch (View)
  float rs1[kBatch], rv1[kBatch];   // stayer results
  float pa[kBatch], plim[kBatch], plimrel[kBatch], pvlim[kBatch];   // pass state
  int pnext1[kBatch];
  uint32_t pfl[kBatch];
  uint8_t tix[kBatch], kind[kBatch];
  uint16_t cand[kBatch], defl[kBatch];
  unsigned long long skh[kInPool];  // inbox keys per tile, sorted
  int skv[kInPool], bs[kInPool];
  int ncand, ndef;
  TileSh T[kMaxT];
  Prof prof[kSmemProf];
};

struct StepSmem {
  Stage S[kStages];
  Cons C;
};

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
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
               : "memory");
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
__device__ __forceinline__ void cbar() {
  asm volatile("bar.sync %0, %1;" ::"r"(kCBar), "r"(kCT) : "memory");
}

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

// A vehicle that leaves its slot: lane change / hand-off (kind 2) or arrival
// (kind 3).  Counters go to the tile's shared-memory accumulators.
__device__ __noinline__ void emit_moved(const StepArgs &A, const View &C, int i, const Res &r,
                                        int kind, TileSh &T) {
  const int vid = C.vid(i);
  if (r.lc != 0) atomicAdd(&T.c_lc, 1);
  if (r.hand) atomicAdd(&T.c_hand, r.hand);
  if (kind == 3) {
    A.status[vid] = ST_FINISHED;
    A.arrive_time[vid] = A.t + 1;
    A.wait_fin[vid] = r.wait1;
    atomicAdd(&T.c_fin, 1);
    long long *ta = A.tacc + (size_t)T.tile * kNAcc;
    red_add(ta + ACC_SUM_TRAVEL, (long long)(A.t + 1 - A.insert_time[vid]));
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
  rec.meta = pack_meta(A.lane_local[r.lane_g], m_prof(meta), r.cursor);
  rec.wait = r.wait1;
  rec.pad = 0;
  const int dt = A.lane_tile[r.lane_g];
  const int owner = A.tile_owner[dt];
  if (owner == A.rank) {
    const int slot = atomicAdd(&A.icnt_out[dt], 1);
    if (slot < A.tile_icap[dt]) put_inbox(A.inbox_out + A.tile_ibase[dt] + slot, rec);
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

// ---- producer warp --------------------------------------------------------------
struct TInfo { int tile, n_st, n_in, base, ibase, cap, icap, doff, dw, nl, nroad; };

__device__ __forceinline__ TInfo load_tinfo(const StepArgs &A, int idx) {
  TInfo x;
  x.tile = -1;
  x.n_st = x.n_in = x.base = x.ibase = x.cap = x.icap = x.doff = x.dw = x.nl = x.nroad = 0;
  if (idx < A.n_own) {
    const int t = A.tiles[idx];
    x.tile = t;
    x.n_st = A.cnt_in[t];
    x.n_in = A.icnt_in[t];
    x.base = A.tile_base[t];
    x.ibase = A.tile_ibase[t];
    x.cap = A.tile_cap[t];
    x.icap = A.tile_icap[t];
    x.doff = A.desc_off[t];
    x.dw = A.desc_off[t + 1] - x.doff;
    x.nl = A.tile_lane_off[t + 1] - A.tile_lane_off[t];
    x.nroad = A.tile_nroad[t];
  }
  return x;
}
__device__ __forceinline__ TInfo shfl_tinfo(const TInfo &x, int src) {
  TInfo y;
  y.tile = __shfl_sync(0xffffffffu, x.tile, src);
  y.n_st = __shfl_sync(0xffffffffu, x.n_st, src);
  y.n_in = __shfl_sync(0xffffffffu, x.n_in, src);
  y.base = __shfl_sync(0xffffffffu, x.base, src);
  y.ibase = __shfl_sync(0xffffffffu, x.ibase, src);
  y.cap = __shfl_sync(0xffffffffu, x.cap, src);
  y.icap = __shfl_sync(0xffffffffu, x.icap, src);
  y.doff = __shfl_sync(0xffffffffu, x.doff, src);
  y.dw = __shfl_sync(0xffffffffu, x.dw, src);
  y.nl = __shfl_sync(0xffffffffu, x.nl, src);
  y.nroad = __shfl_sync(0xffffffffu, x.nroad, src);
  return y;
}

__device__ __noinline__ void producer(const StepArgs &A, StepSmem &M, const Prof *P, int lane) {
  int stage = 0;
  unsigned phase = 0;
  // lanes 0..15 hold the current group of claimed tiles, lanes 16..31 the next
  int gb = 0;
  if (lane == 0) gb = atomicAdd(&A.work[0], kGroup);
  gb = __shfl_sync(0xffffffffu, gb, 0);
  int nb = 0;
  if (lane == 0) nb = atomicAdd(&A.work[0], kGroup);
  nb = __shfl_sync(0xffffffffu, nb, 0);
  TInfo mine = load_tinfo(A, (lane < kGroup ? gb : nb) + (lane & (kGroup - 1)));
  int gpos = 0;
  bool exhausted = false;
  for (;;) {
    Stage &S = M.S[stage];
    BatchHdr &H = S.H;
    mbar_wait(&S.empty, phase ^ 1u);                 // the consumers released the stage
    int nt = 0, nveh = 0, nin = 0, nst = 0, nd = 0, nx = 0, np = 0, sw = 0, gm = 0;
    unsigned tx = 0;
    while (!exhausted) {
      if (gpos == kGroup) {                          // next group: shift and claim another
        TInfo up = shfl_tinfo(mine, (lane + kGroup) & 31);
        int c = 0;
        if (lane == 0) c = atomicAdd(&A.work[0], kGroup);
        c = __shfl_sync(0xffffffffu, c, 0);
        TInfo fresh = load_tinfo(A, c + (lane & (kGroup - 1)));
        mine = lane < kGroup ? up : fresh;
        gpos = 0;
      }
      const TInfo x = shfl_tinfo(mine, gpos);
      if (x.tile < 0) { exhausted = true; break; }
      const int n = x.n_st + x.n_in, r4 = (x.n_st + 3) & ~3, nj = x.nl - x.nroad;
      const bool big = n > kBatch || x.n_in > kInPool || x.dw > kDescPool || nj > kXPool ||
                       x.nroad > kPPool || 7 * r4 > kSlabWords;
      if (big && nt > 0) break;                      // a large tile goes alone (global mode)
      if (!big && (nt == kMaxT || nveh + n > kBatch || nin + x.n_in > kInPool || nd + x.dw > kDescPool ||
                   nx + nj > kXPool || np + x.nroad > kPPool || sw + 7 * r4 > kSlabWords))
        break;
      if (lane == 0) {
        H.tile[nt] = x.tile; H.n_st[nt] = x.n_st; H.n_in[nt] = x.n_in; H.base[nt] = x.base;
        H.ibase[nt] = x.ibase; H.cap[nt] = x.cap; H.icap[nt] = x.icap; H.nl[nt] = x.nl;
        H.nroad[nt] = x.nroad; H.doff[nt] = x.doff; H.dw[nt] = x.dw;
        H.slab[nt] = sw; H.r4[nt] = r4; H.in0[nt] = nin; H.st0[nt] = nst; H.desc[nt] = nd;
        H.xo[nt] = nx; H.po[nt] = np; H.snap0[nt] = nveh;
      }
      if (!big) {
        tx += (x.n_st > 0 ? 7u * 4u * (unsigned)r4 : 0u) + 32u * (unsigned)x.n_in + 4u * (unsigned)x.dw;
        sw += 7 * r4;
        nin += x.n_in;
        nd += x.dw;
      }
      nt += 1;
      nveh += n;
      nst += x.n_st;
      nx += nj;
      np += x.nroad;
      gpos += 1;
      if (big) { gm = 1; break; }
    }
    if (lane == 0) {
      H.nt = nt; H.gmode = gm; H.done = nt == 0; H.nveh = nveh; H.nst = nst; H.nin = nin;
      mbar_arrive_tx(&S.full, gm ? 0u : tx);
    }
    __syncwarp();
    if (nt == 0) {                                   // no more work: tell the consumers
      if (lane == 0) mbar_arrive(&S.full);
      break;
    }
    if (!gm && lane < nt) {                          // bulk copies of tile `lane`
      const int k = lane;
      const int ns = H.n_st[k], ni = H.n_in[k], b0 = H.base[k], r4 = H.r4[k];
      if (ns > 0) {
        uint32_t *d = S.slab + H.slab[k];
        const unsigned by = 4u * (unsigned)r4;
        bulk_g2s(d + 0 * r4, A.in.s + b0, by, &S.full);
        bulk_g2s(d + 1 * r4, A.in.v + b0, by, &S.full);
        bulk_g2s(d + 2 * r4, A.in.vid + b0, by, &S.full);
        bulk_g2s(d + 3 * r4, A.in.nxt + b0, by, &S.full);
        bulk_g2s(d + 4 * r4, A.in.nxt2 + b0, by, &S.full);
        bulk_g2s(d + 5 * r4, A.in.meta + b0, by, &S.full);
        bulk_g2s(d + 6 * r4, A.in.wait + b0, by, &S.full);
      }
      if (ni > 0) bulk_g2s(S.inbox + H.in0[k], A.inbox_in + H.ibase[k], 32u * (unsigned)ni, &S.full);
      bulk_g2s(S.desc + H.desc[k], A.desc + H.doff[k], 4u * (unsigned)H.dw[k], &S.full);
    }
    // gathers (global loads, off the consumers' critical path): per junction
    // lane its signal at t and the first vehicle of its exit lane at t
    for (int q = lane; q < nx; q += 32) {
      int k = 0;
      while (k + 1 < nt && H.xo[k + 1] <= q) ++k;
      const int nl = H.nl[k], l = H.nroad[k] + (q - H.xo[k]);
      const int *W = A.desc + H.doff[k];
      const int g = W[4 + l], b = W[4 + 4 * nl + l];
      ExtFirst e;
      e.sig = A.lane_sig[g];
      e.b = b;
      e.Lb = A.lane_len[b];
      e.pad = 0;
      unsigned long long key;
      const float *pv = A.pubv_cur;
      if (!A.peers) {
        key = A.summ_cur[b];
      } else {
        const int bt = A.lane_tile[b];
        const int ow = A.tile_owner[bt];
        if (ow == A.rank) key = A.summ_cur[b];
        else key = peer_summary(A, bt, b, pv);
      }
      e.vid = -1;
      e.s = e.v = e.len = 0.f;
      if (key != kEmptyKey) {
        e.vid = (int)(unsigned)(key & 0xffffffffu);
        e.s = __uint_as_float((unsigned)(key >> 32));
        e.v = pv[e.vid];
        e.len = P[A.veh_prof[e.vid]].len;
      }
      S.ext[q] = e;
    }
    // heads of the pending-departure queues of the road lanes (K11)
    for (int q = lane; q < np; q += 32) {
      int k = 0;
      while (k + 1 < nt && H.po[k + 1] <= q) ++k;
      const int l = q - H.po[k];
      const int g = A.desc[H.doff[k] + 4 + l];
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
        if (dep <= A.t) {
          ph.k = vk;
          ph.depart = dep;
          ph.start_s = A.start_s[vk];
          ph.prof = A.veh_prof[vk];
        }
      }
      S.pend[q] = ph;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.full);
    stage += 1;
    if (stage == kStages) { stage = 0; phase ^= 1u; }
  }
}

// ---- consumer phases ------------------------------------------------------------
// Tile metadata from its descriptor into shared memory (one warp).
__device__ __forceinline__ void tile_setup(const StepArgs &A, const BatchHdr &H, int k,
                                           const int *W, const ExtFirst *ext, const PendHead *pend,
                                           const Prof *P, TileSh &T, int lane_id) {
  const int nl = H.nl[k], nroad = H.nroad[k];
  const int ne = W[2];
  const int eo = 4 + 5 * nl + 6 * nroad;
  if (lane_id == 0) {
    T.nl = nl;
    T.nroad = nroad;
    T.tile = H.tile[k];
    T.base = H.base[k];
    T.ibase = H.ibase[k];
    T.cap = H.cap[k];
    T.icap = H.icap[k];
    T.snap0 = H.snap0[k];
    T.n = H.n_st[k] + H.n_in[k];
    T.P = P;
    T.ext = ext;
    T.pend = pend;
    T.run = 0;
    T.c_fin = T.c_lc = T.c_hand = T.c_guard = T.c_ovf = T.c_ins = 0;
    T.c_delay = 0ull;
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
  if (lane_id < ne) {
    const int *ew = W + eo + 8 * lane_id;
    const unsigned fl = (unsigned)ew[3];
    const int jl = (int)(fl >> 24);
    SuccEnt e;
    e.j = ew[0];
    e.troad = ew[1];
    e.b = ew[2];
    e.outr = make_int4(ew[4], ew[5], ew[6], ew[7]);
    const bool stop = (fl & 1u) && ext[jl - nroad].sig != SIG_GREEN;
    e.fl = (stop ? 1 : 0) | ((int)(jl & 0xff) << 8);
    T.se[(fl >> 8) & 0xff][(fl >> 16) & 0xff] = e;
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
#pragma unroll 1
    for (int q = 0; q < kMaxRoadLanes * kMaxGroups; ++q) {
      const int Rq = __shfl_sync(0xffffffffu, R, q);
      if (valid && ((vb >> q) & 1u) && Rq == R && q < lane_id) first = false;
    }
    const unsigned fb = __ballot_sync(0xffffffffu, first);
#pragma unroll 1
    for (int q = 0; q < kMaxRoadLanes * kMaxGroups; ++q) {
      const int Rq = __shfl_sync(0xffffffffu, R, q);
      if (valid && ((fb >> q) & 1u) && Rq == R) myk = __popc(fb & ((1u << q) - 1u));
    }
    if (first) T.troad[myk] = R;
    if (valid) T.gidx[a][myk] = (int8_t)g;
    const int ntr = __popc(fb);
    for (int kk = 0; kk < ntr; ++kk) {
      const unsigned m = __ballot_sync(0xffffffffu, valid && myk == kk);
      unsigned lanes = 0;
#pragma unroll
      for (int aa = 0; aa < kMaxRoadLanes; ++aa)
        if ((m >> (aa * kMaxGroups)) & ((1u << kMaxGroups) - 1u)) lanes |= 1u << aa;
      if (lane_id == 0) T.reach[kk] = (uint8_t)lanes;
    }
    const unsigned um = __ballot_sync(0xffffffffu, lane_id < nroad && T.usable[lane_id]);
    if (lane_id == 0) { T.ntr = ntr; T.umask = um; }
  }
}

// tile of a flat index given per-tile starts (nt <= kMaxT, ascending)
__device__ __forceinline__ int find_tile(const int *start, int nt, int f) {
  int k = 0;
  while (k + 1 < nt && start[k + 1] <= f) ++k;
  return k;
}

// warp-aggregated append to a shared list
__device__ __forceinline__ void push_list(bool pred, uint16_t *list, int *count, int val) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  const int leader = __ffs(m) - 1;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)val;
}

// the vehicle at snapshot slot i has been updated (fp32 path or fp64
// canonical path): stayer results stay in shared memory for the in-order
// compaction, movers and arrivals leave now
__device__ __forceinline__ void settle(const StepArgs &A, Cons &K, const View &C, int i, int li,
                                       const Res &r, TileSh &T) {
  const int l = m_lane(C.meta(i));
  if (r.fin) {
    emit_moved(A, C, i, r, 3, T);
    K.kind[li] = 3;
  } else if (r.lc == 0 && r.hand == 0 && r.lane_g == T.glob[l]) {
    K.rs1[li] = r.s1;
    K.rv1[li] = r.v1;
    C.wait(i) = r.wait1;
    K.kind[li] = 1;
  } else {
    emit_moved(A, C, i, r, 2, T);
    K.kind[li] = 2;
  }
}

// pass 1: lane-change eligibility and O4-O6 on the current lane (fp32)
__device__ __forceinline__ void pass1(const StepArgs &A, Cons &K, const View &C, int i, int li,
                                      const TileSh &T) {
  const uint32_t meta = C.meta(i);
  const int l = m_lane(meta);
  Me me;
  me.vid = C.vid(i);
  me.cur = m_cursor(meta);
  me.nxt = C.nxt(i);
  me.nxt2 = C.nxt2(i);
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
  g.why = 0;
  Elig E;
  E.sl0 = E.sl1 = -1;
  E.mand = 0;
  E.inG = true;
  E.want0 = E.want1 = false;
  me.k = -1;
  if (T.isroad[l]) E = lc_elig<float, true>(A, T, l, s, v, p, me, g);
  const LEv<float> use = eval_lane<float, true>(A, T, C, l, lead, s, v, p, me, g);
  if (A.record) {
    A.r_leader[me.vid] = use.leader;
    A.r_hops[me.vid] = (int8_t)use.hops;
    A.r_phantom[me.vid] = (int8_t)use.phantom;
  }
  K.pa[li] = use.a;
  K.plim[li] = use.lim;
  K.plimrel[li] = use.limrel;
  K.pvlim[li] = use.vlim;
  K.pnext1[li] = use.next1;
  K.pfl[li] = (use.has_lim ? F_LIM : 0u) | (g.hit ? F_HIT : 0u) | (E.inG ? F_ING : 0u) |
              (E.want0 ? F_W0 : 0u) | (E.want1 ? F_W1 : 0u) | ((uint32_t)(E.mand + 1) << F_MAND_SH) |
              ((uint32_t)(me.k + 1) << F_K_SH) | ((uint32_t)l << F_NL_SH) | (1u << F_LC_SH);
}

// pass 2: O7 (MOBIL) for a vehicle that may change lane (fp32)
__device__ __forceinline__ void pass2(const StepArgs &A, Cons &K, const View &C, int i, int li,
                                      const TileSh &T) {
  const uint32_t meta = C.meta(i);
  const int l = m_lane(meta);
  const uint32_t fl = K.pfl[li];
  Me me;
  me.vid = C.vid(i);
  me.cur = m_cursor(meta);
  me.nxt = C.nxt(i);
  me.nxt2 = C.nxt2(i);
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
  g.why = 0;
  const SideRes<float> sr = lc_decide<float, true>(A, T, C, i, l, s, v, p, me, E, K.pa[li], g);
  if (g.hit) {
    K.pfl[li] = fl | F_HIT;
  } else if (sr.choice >= 0) {
    K.pa[li] = sr.a;
    K.plim[li] = sr.lim;
    K.plimrel[li] = sr.limrel;
    K.pvlim[li] = sr.vlim;
    K.pnext1[li] = sr.next1;
    const int nl = sr.choice == 0 ? E.sl0 : E.sl1;
    const int lc = sr.choice == 0 ? -1 : 1;
    K.pfl[li] = (fl & ~(F_LIM | (0xffu << F_NL_SH) | (3u << F_LC_SH))) | (sr.has_lim ? F_LIM : 0u) |
                ((uint32_t)nl << F_NL_SH) | ((uint32_t)(lc + 1) << F_LC_SH);
  }
}

// pass 3: O8-O9 (fp32).  Returns false if the vehicle must be recomputed.
__device__ __forceinline__ bool pass3(const StepArgs &A, Cons &K, const View &C, int i, int li,
                                      TileSh &T) {
  const uint32_t fl = K.pfl[li];
  if (fl & F_HIT) return false;
  const uint32_t meta = C.meta(i);
  Me me;
  me.vid = C.vid(i);
  me.cur = m_cursor(meta);
  me.nxt = C.nxt(i);
  me.nxt2 = C.nxt2(i);
  me.k = -1;
  LEv<float> use;
  use.a = K.pa[li];
  use.lim = K.plim[li];
  use.limrel = K.plimrel[li];
  use.vlim = K.pvlim[li];
  use.next1 = K.pnext1[li];
  use.has_lim = (fl & F_LIM) != 0;
  const int new_l = (int)((fl >> F_NL_SH) & 0xffu);
  const int lc = (int)((fl >> F_LC_SH) & 3u) - 1;
  Guard g;
  g.hit = false;
  g.why = 0;
  Res r;
  integrate<float, true>(A, T, C.s(i), C.v(i), me, use, lc, new_l, C.wait(i), r, g);
  if (g.hit) return false;
  if (A.record) record(A, me.vid, r, false);
  settle(A, K, C, i, li, r, T);
  return true;
}

// the fp64 canonical recomputation of one vehicle
__device__ __noinline__ void pass_fp64(const StepArgs &A, Cons &K, const View &C, int i, int li,
                                       TileSh &T) {
  Res r;
  Guard g;
  g.hit = false;
  g.why = 0;
  veh_update<double, false>(A, T, C, i, r, g);
  if (A.record) record(A, C.vid(i), r, true);
  settle(A, K, C, i, li, r, T);
}

// In-order compaction of the stayers of snapshot range [a, b) of tile T (one
// warp): each goes to the tile's slab at base + run (coalesced), the first
// stayer of each lane is remembered for the t+1 summary.
__device__ __forceinline__ void compact(const StepArgs &A, Cons &K, const View &C, TileSh &T, int a,
                                        int b, int c0, int lane_id) {
  int run = T.run;
  for (int i0 = a; i0 < b; i0 += 32) {
    const int i = i0 + lane_id;
    const bool st = i < b && K.kind[i - c0] == 1;
    const unsigned ball = __ballot_sync(0xffffffffu, st);
    if (st) {
      const int rank = run + __popc(ball & ((1u << lane_id) - 1u));
      if (rank < T.cap) {
        const int pos = T.base + rank;
        const uint32_t meta = C.meta(i);
        A.out.s[pos] = K.rs1[i - c0];
        A.out.v[pos] = K.rv1[i - c0];
        A.out.vid[pos] = C.vid(i);
        A.out.nxt[pos] = C.nxt(i);
        A.out.nxt2[pos] = C.nxt2(i);
        A.out.meta[pos] = meta;
        A.out.wait[pos] = C.wait(i);
        atomicMin(&T.first_out[m_lane(meta)], (rank << 15) | (i - T.snap0));
      } else {
        atomicAdd(&T.c_ovf, 1);                     // slab capacity exceeded: sticky SIM_E_CAPACITY
      }
    }
    run += __popc(ball);
  }
  __syncwarp();
  if (lane_id == 0) T.run = run;
  __syncwarp();
}

// Lane summaries for t+1, departures (K11; L25) and counters (a6) of
// one tile (one warp), after all its vehicles are settled.
__device__ __forceinline__ void tile_finish(const StepArgs &A, Cons &K, const View &C, TileSh &T,
                                            bool gmode, int lane_id) {
  const int nl = T.nl, nroad = T.nroad, tile = T.tile;
  const int run = T.run < T.cap ? T.run : T.cap;
  for (int l = lane_id; l < nl; l += 32) {
    const int g = T.glob[l];
    const int fo = T.first_out[l];
    if (fo != 0x7fffffff) {
      const int rank = fo >> 15, idx = T.snap0 + (fo & 0x7fff);
      const int vid = C.vid(idx);
      float s1, v1;
      if (!gmode) { s1 = K.rs1[idx]; v1 = K.rv1[idx]; }
      else { s1 = A.out.s[T.base + rank]; v1 = A.out.v[T.base + rank]; }
      atomicMin(&A.summ_next[g], vkey(s1, vid));
      A.pubv_next[vid] = v1;
      if (A.lane_cnt_next) {                          // stayers of lane l: [rank, next lane's first)
        int end = run;
        for (int q = l + 1; q < nl; ++q)
          if (T.first_out[q] != 0x7fffffff) { end = T.first_out[q] >> 15; break; }
        atomicAdd(&A.lane_cnt_next[g], end - rank);
      }
    }
    A.summ_clear[g] = kEmptyKey;
  }
  for (int l = lane_id; l < nroad; l += 32) {         // departures (K11; ledger L25)
    const PendHead ph = T.pend[l];
    if (ph.k < 0 || !T.usable[l]) continue;
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
    if (!ok) continue;
    InboxRec rec;
    rec.s = (float)ss;
    rec.v = 0.f;
    rec.vid = k;
    const int off = A.route_start[k], rl = A.route_len[k];
    rec.nxt = rl > 1 ? A.route[off + 1] : -1;
    rec.nxt2 = rl > 2 ? A.route[off + 2] : -1;
    rec.meta = pack_meta(l, ph.prof, 0);
    rec.wait = 0;
    rec.pad = 0;
    const int slot = atomicAdd(&A.icnt_out[tile], 1);
    if (slot < T.icap) put_inbox(A.inbox_out + T.ibase + slot, rec);
    else atomicAdd(&T.c_ovf, 1);
    atomicMin(&A.summ_next[g], vkey(rec.s, k));
    A.pubv_next[k] = 0.f;
    if (A.lane_cnt_next) atomicAdd(&A.lane_cnt_next[g], 1);
    A.pend_head[g] = ph.h + 1;
    A.status[k] = ST_DRIVING;
    A.insert_time[k] = A.t + 1;
    if (A.record) A.r_ins[k] = 1;
    atomicAdd(&T.c_ins, 1);
    atomicAdd(&T.c_delay, (unsigned long long)(long long)(A.t + 1 - ph.depart));
  }
  __syncwarp();
  if (lane_id == 0) {
    long long *ta = A.tacc + (size_t)tile * kNAcc;
    red_add(ta + ACC_VEH_STEPS, T.n);
    if (T.c_fin) red_add(ta + ACC_FINISHED, T.c_fin);
    if (T.c_ins) {
      red_add(ta + ACC_INSERTED, T.c_ins);
      red_add(ta + ACC_SUM_DELAY, (long long)T.c_delay);
    }
    if (T.c_lc) red_add(ta + ACC_LANE_CHANGES, T.c_lc);
    if (T.c_hand) red_add(ta + ACC_HANDOFFS, T.c_hand);
    if (T.c_guard) red_add(ta + ACC_GUARD, T.c_guard);
    if (T.c_ovf) red_add(ta + ACC_OVERFLOW, T.c_ovf);
    A.cnt_out[tile] = run;
    A.icnt_in[tile] = 0;
  }
}

// passes 1-3 and the fp64 recomputation over snapshot slots [c0, c1)
template <bool EXACT>
__device__ __forceinline__ void run_passes(const StepArgs &A, Cons &K, const View &C, int c0, int c1,
                                           bool gm, int tid) {
  const int n = c1 - c0;
  if (tid == 0) { K.ncand = 0; K.ndef = 0; }
  cbar();
  if constexpr (!EXACT) {
    for (int q0 = 0; q0 < n; q0 += kCT) {            // pass 1 (every vehicle)
      const int q = q0 + tid;
      bool cand = false;
      if (q < n) {
        const int i = c0 + q;
        const TileSh &T = K.T[gm ? 0 : K.tix[q]];
        pass1(A, K, C, i, q, T);
        const uint32_t fl = K.pfl[q];
        const int l = m_lane(C.meta(i));
        cand = !(fl & F_HIT) && ((fl & (F_W0 | F_W1)) || (A.record && T.isroad[l]));
      }
      push_list(cand, K.cand, &K.ncand, q);
    }
    cbar();
    const int nc = K.ncand;
    for (int q = tid; q < nc; q += kCT) {            // pass 2 (compacted MOBIL candidates)
      const int li = K.cand[q];
      pass2(A, K, C, c0 + li, li, K.T[gm ? 0 : K.tix[li]]);
    }
    cbar();
    for (int q0 = 0; q0 < n; q0 += kCT) {            // pass 3 (every vehicle)
      const int q = q0 + tid;
      bool def = false;
      if (q < n) def = !pass3(A, K, C, c0 + q, q, K.T[gm ? 0 : K.tix[q]]);
      push_list(def, K.defl, &K.ndef, q);
    }
    cbar();
  } else {
    for (int q = tid; q < n; q += kCT) K.defl[q] = (uint16_t)q;
    if (tid == 0) K.ndef = n;
    cbar();
  }
  const int nd = K.ndef;
  for (int q = tid; q < nd; q += kCT) {              // fp64 canonical path
    const int li = K.defl[q];
    TileSh &T = K.T[gm ? 0 : K.tix[li]];
    pass_fp64(A, K, C, c0 + li, li, T);
    if (!EXACT) atomicAdd(&T.c_guard, 1);
  }
  cbar();
}

template <bool EXACT>
__device__ __forceinline__ void consumer(const StepArgs &A, StepSmem &M, const Prof *P, int tid) {
  Cons &K = M.C;
  const int warp = tid >> 5, lane_id = tid & 31;
  int stage = 0;
  unsigned phase = 0;
  for (;;) {
    Stage &S = M.S[stage];
    mbar_wait(&S.full, phase);
    const BatchHdr &H = S.H;
    if (H.done) break;
    const int nt = H.nt;
    const bool gm = H.gmode != 0;
    View C;
    if (!gm) {
      C.p = K.snap;
      C.st = kBatch;
    } else {
      C.st = H.cap[0] + H.icap[0];
      C.p = A.scratch + 7 * (size_t)(H.base[0] + H.ibase[0]);
    }
    // ---- A: tile metadata (warp per tile) + inbox ranks (flat) -----------------
    for (int k = warp; k < nt; k += kCW) {
      const int *W = gm ? A.desc + H.doff[k] : S.desc + H.desc[k];
      tile_setup(A, H, k, W, S.ext + H.xo[k], S.pend + H.po[k], P, K.T[k], lane_id);
    }
    if (!gm) {
      for (int r = tid; r < H.nin; r += kCT) {
        const int k = find_tile(H.in0, nt, r);
        const int a = H.in0[k], ni = H.n_in[k];
        const InboxRec &x = S.inbox[r];
        const unsigned long long h = hikey(m_lane(x.meta), x.s);
        int rank = 0;
        for (int q = 0; q < ni; ++q) {
          const InboxRec &o = S.inbox[a + q];
          rank += key_less(hikey(m_lane(o.meta), o.s), o.vid, h, x.vid);
        }
        K.skh[a + rank] = h;
        K.skv[a + rank] = x.vid;
        K.bs[a + rank] = r - a;
      }
    } else if (H.n_in[0] > 0) {
      rank_inbox_global(A.inbox_in + H.ibase[0], H.n_in[0], A.bsort_scratch + H.ibase[0], tid, kCT);
    }
    cbar();
    // ---- B: merge stayers + sorted inbox into the snapshot (a1) ----------------
    if (!gm) {
      for (int f = tid; f < H.nst; f += kCT) {        // stayers
        const int k = find_tile(H.st0, nt, f);
        const int i = f - H.st0[k], r4 = H.r4[k];
        const uint32_t *sl = S.slab + H.slab[k];
        const float s = __uint_as_float(sl[i]);
        const uint32_t meta = sl[5 * r4 + i];
        const int vid = (int)sl[2 * r4 + i];
        const int a = H.in0[k], ni = H.n_in[k];
        int lo = 0, hi = ni;
        if (ni > 0) {
          const unsigned long long h = hikey(m_lane(meta), s);
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (key_less(K.skh[a + mid], K.skv[a + mid], h, vid)) lo = mid + 1; else hi = mid;
          }
        }
        const int pos = H.snap0[k] + i + lo;
        C.s(pos) = s;
        C.v(pos) = __uint_as_float(sl[r4 + i]);
        C.vid(pos) = vid;
        C.meta(pos) = meta;
        C.nxt(pos) = (int)sl[3 * r4 + i];
        C.nxt2(pos) = (int)sl[4 * r4 + i];
        C.wait(pos) = (int)sl[6 * r4 + i];
        K.tix[pos] = (uint8_t)k;
      }
      for (int r = tid; r < H.nin; r += kCT) {        // inbox records
        const int k = find_tile(H.in0, nt, r);
        const int a = H.in0[k], rank = r - a, ns = H.n_st[k], r4 = H.r4[k];
        const InboxRec &x = S.inbox[a + K.bs[r]];
        const unsigned long long h = hikey(m_lane(x.meta), x.s);
        const uint32_t *sl = S.slab + H.slab[k];
        int lo = 0, hi = ns;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (key_less(hikey(m_lane(sl[5 * r4 + mid]), __uint_as_float(sl[mid])), (int)sl[2 * r4 + mid], h,
                       x.vid))
            lo = mid + 1;
          else
            hi = mid;
        }
        const int pos = H.snap0[k] + rank + lo;
        C.s(pos) = x.s;
        C.v(pos) = x.v;
        C.vid(pos) = x.vid;
        C.meta(pos) = x.meta;
        C.nxt(pos) = x.nxt;
        C.nxt2(pos) = x.nxt2;
        C.wait(pos) = x.wait;
        K.tix[pos] = (uint8_t)k;
      }
    } else {
      const int ns = H.n_st[0], ni = H.n_in[0], base = H.base[0], ib = H.ibase[0];
      const InboxRec *inb = A.inbox_in + ib;
      const int *bsort = A.bsort_scratch + ib;
      for (int i = tid; i < ns; i += kCT) {
        const int gi = base + i;
        const float s = A.in.s[gi];
        const uint32_t meta = A.in.meta[gi];
        const int vid = A.in.vid[gi];
        const int lo = ni > 0 ? lower_bound_inbox_global(inb, bsort, ni, hikey(m_lane(meta), s), vid) : 0;
        const int pos = i + lo;
        C.s(pos) = s;
        C.v(pos) = A.in.v[gi];
        C.vid(pos) = vid;
        C.meta(pos) = meta;
        C.nxt(pos) = A.in.nxt[gi];
        C.nxt2(pos) = A.in.nxt2[gi];
        C.wait(pos) = A.in.wait[gi];
      }
      for (int r = tid; r < ni; r += kCT) {
        const InboxRec x = inb[bsort[r]];
        const unsigned long long h = hikey(m_lane(x.meta), x.s);
        int lo = 0, hi = ns;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const int gi = base + mid;
          if (key_less(hikey(m_lane(A.in.meta[gi]), A.in.s[gi]), A.in.vid[gi], h, x.vid)) lo = mid + 1;
          else hi = mid;
        }
        const int pos = r + lo;
        C.s(pos) = x.s;
        C.v(pos) = x.v;
        C.vid(pos) = x.vid;
        C.meta(pos) = x.meta;
        C.nxt(pos) = x.nxt;
        C.nxt2(pos) = x.nxt2;
        C.wait(pos) = x.wait;
      }
    }
    cbar();
    // ---- C: lane segments of the snapshot ---------------------------------------
    const int nveh = H.nveh;
    for (int i = tid; i < nveh; i += kCT) {
      const int k = gm ? 0 : K.tix[i];
      TileSh &T = K.T[k];
      const int l = m_lane(C.meta(i));
      if (i == T.snap0 || m_lane(C.meta(i - 1)) != l) T.seg_start[l] = (int16_t)i;
      if (i == T.snap0 + T.n - 1 || m_lane(C.meta(i + 1)) != l) T.seg_end[l] = (int16_t)(i + 1);
    }
    cbar();
    // ---- D-G: the vehicle passes; H: compaction and per-tile finish -------------
    if (!gm) {
      run_passes<EXACT>(A, K, C, 0, nveh, false, tid);
      for (int k = warp; k < nt; k += kCW) {
        TileSh &T = K.T[k];
        compact(A, K, C, T, T.snap0, T.snap0 + T.n, 0, lane_id);
        tile_finish(A, K, C, T, false, lane_id);
      }
    } else {
      for (int c0 = 0; c0 < nveh; c0 += kBatch) {
        const int c1 = min(nveh, c0 + kBatch);
        run_passes<EXACT>(A, K, C, c0, c1, true, tid);
        if (warp == 0) compact(A, K, C, K.T[0], c0, c1, c0, lane_id);
        cbar();
      }
      if (warp == 0) tile_finish(A, K, C, K.T[0], true, lane_id);
    }
    cbar();
    if (tid == 0) mbar_arrive(&S.empty);             // the stage can be refilled
    stage += 1;
    if (stage == kStages) { stage = 0; phase ^= 1u; }
  }
}

template <bool EXACT>
__global__ void __launch_bounds__(kStepThreads, 2) k_step(const __grid_constant__ StepArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  StepSmem &M = *reinterpret_cast<StepSmem *>(smem_raw);
  const int tid = threadIdx.x;
  const Prof *P = A.prof;
  if (A.n_prof <= kSmemProf) {                      // profiles as int4 words (Prof is 96 B)
    const int nw = A.n_prof * (int)(sizeof(Prof) / 16);
    for (int q = tid; q < nw; q += blockDim.x)
      reinterpret_cast<int4 *>(M.C.prof)[q] = reinterpret_cast<const int4 *>(A.prof)[q];
    P = M.C.prof;
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&M.S[s].full, 2);
      mbar_init(&M.S[s].empty, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= kCT) producer(A, M, P, tid & 31);
  else consumer<EXACT>(A, M, P, tid);
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&A.work[1], 1) == (int)gridDim.x - 1) {
      A.work[0] = 0;
      A.work[1] = 0;
    }
  }
}

int step_smem_bytes() { return (int)sizeof(StepSmem); }

void launch_step(const StepArgs &a, void *stream, int smem_bytes) {
  static int resident[2] = {0, 0};                  // resident blocks per GPU, per instantiation
  if (!resident[0]) {
    cudaFuncSetAttribute(k_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    int dev = 0, nsm = 0, b0 = 0, b1 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, k_step<false>, kStepThreads, smem_bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_step<true>, kStepThreads, smem_bytes);
    resident[0] = std::max(1, b0) * std::max(1, nsm);
    resident[1] = std::max(1, b1) * std::max(1, nsm);
  }
  if (a.n_own <= 0) return;
  const int ex = a.exact_mode ? 1 : 0;
  // enough CTAs for the work (a CTA takes kGroup tiles at a time), at most
  // the resident capacity (persistent)
  const int grid = std::min((a.n_own + kGroup - 1) / kGroup, resident[ex]);
  if (ex) k_step<true><<<grid, kStepThreads, smem_bytes, (cudaStream_t)stream>>>(a);
  else k_step<false><<<grid, kStepThreads, smem_bytes, (cudaStream_t)stream>>>(a);
}

}  // namespace sim
