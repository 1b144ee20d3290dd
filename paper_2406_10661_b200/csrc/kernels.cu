// kernels.cu — the signal kernel (a5) and the read-side / exchange kernels.
// The fused step kernel k_step (a0-a4, a6) is in kstep.cu.
#include <cuda_runtime.h>

#include <algorithm>

#include "dev.h"
#include "model.cuh"

namespace sim {

__device__ __forceinline__ unsigned long long vkey(float s, int vid) {
  return ((unsigned long long)__float_as_uint(s) << 32) | (unsigned)vid;
}

__device__ __forceinline__ void put_inbox(InboxRec *dst, const InboxRec &rec) {
  int4 *d = reinterpret_cast<int4 *>(dst);
  const int4 *s = reinterpret_cast<const int4 *>(&rec);
  d[0] = s[0];
  d[1] = s[1];
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
  pdl_wait();                                       // the lane counts of t (previous k_step)
  pdl_trigger();
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
  // (nv > 0; the library passes 0)
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

// Per-group metrics (batched environments), per group: the counters of every
// tile (a tile's rows stay with the partition that accumulated them, also
// after sim_repartition — as in k_reduce_acc) and the driving counts of the
// own tiles.  out [n_groups][kNAcc + 1] (zeroed by the caller).
__global__ void k_reduce_groups(const long long *tacc, int n_tiles, const int32_t *tiles, int n_own,
                                const int32_t *tile_group, const int32_t *cnt,
                                const int32_t *icnt, long long *out) {
  const int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += stride) {
    long long *o = out + (size_t)tile_group[t] * (kNAcc + 1);
    for (int c = 0; c < kNAcc; ++c) {
      const long long x = tacc[(size_t)t * kNAcc + c];
      if (x) atomicAdd(reinterpret_cast<unsigned long long *>(o + c), (unsigned long long)x);
    }
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_own; i += stride) {
    const int t = tiles[i];
    const int d = cnt[t] + icnt[t];
    if (d) atomicAdd(reinterpret_cast<unsigned long long *>(out + (size_t)tile_group[t] * (kNAcc + 1) + kNAcc),
                     (unsigned long long)d);
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
  const InboxRec *rec = tile_recs(A, tile, ns);    // stayers then inbox, contiguous
  for (int i = lane; i < ns + ni; i += 32) {
    const InboxRec r = rec[i];
    const float s = r.s, v = r.v;
    const uint32_t meta = r.meta;
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
    if (slot < A.tile_icap[dt]) put_inbox(A.vout + A.tile_ibase[dt] + slot, m.rec);
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
  const int par = step_t(A) & 1, s3 = step_t(A) % 3;
  const int n = A.cnt_in[T], m = A.icnt_in[T];
  const int base = A.tile_base[T];
  // stayers and inbox records: one contiguous range at the same positions
  const int r0 = base + A.tile_cap[T] - n;
  for (int i = threadIdx.x; i < n + m; i += blockDim.x) {
    const InboxRec r = A.vin[r0 + i];
    put_inbox(Q.inbox[par] + r0 + i, r);
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
    A.cnt_in[T] = 0;                               // the old owner's counts of T at both parities,
    A.icnt_in[T] = 0;                              // so no later read sums a stale count of T
    A.cnt_out[T] = 0;
    A.icnt_out[T] = 0;
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
void launch_signal(const SignalArgs &a, void *stream) {
  if (a.n_junctions > 0)
    launch_pdl(k_signal, dim3((a.n_junctions + 3) / 4), dim3(128), 0, (cudaStream_t)stream, a);
}

// the first step of a captured step graph, written before each replay
__global__ void k_set_i32(int32_t *p, int32_t v) { *p = v; }
void launch_set_i32(int32_t *p, int32_t v, void *stream) { k_set_i32<<<1, 1, 0, (cudaStream_t)stream>>>(p, v); }

void launch_apply_requests(int32_t *request, const int32_t *junc, const int32_t *phase, int m,
                           void *stream) {
  if (m > 0) k_apply_requests<<<(m + 255) / 256, 256, 0, (cudaStream_t)stream>>>(request, junc, phase, m);
}

void launch_reduce_acc(const long long *tacc, int n_tiles, const int32_t *cnt,
                       const int32_t *icnt, const uint8_t *status, int nv, long long *out,
                       void *stream) {
  cudaMemsetAsync(out, 0, (kNAcc + 3) * sizeof(long long), (cudaStream_t)stream);
  k_reduce_acc<<<296, 256, 0, (cudaStream_t)stream>>>(tacc, n_tiles, cnt, icnt, status, nv, out);
}

// ---- sim_read_state_device: the vid-indexed state into caller device buffers ----
// pass 0 (every vid): PENDING defaults; pass 1 (per partition, every vid): the
// latest insert time, FINISHED records; pass 2 (per partition, own tiles): the
// DRIVING vehicles from the tile records (stayers + inbox) — the same merge
// as the host read (sim_read_state), without leaving the device.
__global__ void k_state_defaults(int nv, uint8_t *status, int32_t *lane, int32_t *cursor, int32_t *wait,
                                 int32_t *ins, int32_t *arr, float *s, float *v) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nv) return;
  status[k] = ST_PENDING; lane[k] = -1; cursor[k] = 0; wait[k] = 0; ins[k] = -1; arr[k] = -1;
  s[k] = 0.f; v[k] = 0.f;
}
__global__ void k_state_cold(const StepArgs A, int nv, uint8_t *status, int32_t *wait, int32_t *ins,
                             int32_t *arr) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nv) return;
  atomicMax(&ins[k], A.insert_time[k]);
  if (A.status[k] == ST_FINISHED) { status[k] = ST_FINISHED; arr[k] = A.arrive_time[k]; wait[k] = A.wait_fin[k]; }
}
__global__ void k_state_driving(const StepArgs A, uint8_t *status, int32_t *lane, int32_t *cursor,
                                int32_t *wait, float *s, float *v) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), ln = threadIdx.x & 31;
  if (w >= A.n_own) return;
  const int T = A.tiles[w];
  const int n = A.cnt_in[T] + A.icnt_in[T];
  const InboxRec *rec = tile_recs(A, T, A.cnt_in[T]);
  const int l0 = A.tile_lane_off[T];
  for (int i = ln; i < n; i += 32) {
    const InboxRec r = rec[i];
    status[r.vid] = ST_DRIVING;
    lane[r.vid] = A.tile_lanes[l0 + m_lane(r.meta)];
    cursor[r.vid] = m_cursor(r.meta);
    wait[r.vid] = r.wait;
    s[r.vid] = r.s;
    v[r.vid] = r.v;
  }
}
void launch_state_device(const StepArgs *parts, int n_parts, int nv, uint8_t *status, int32_t *lane,
                         int32_t *cursor, int32_t *wait, int32_t *ins, int32_t *arr, float *s, float *v,
                         void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int g = (nv + 255) / 256;
  if (nv > 0) k_state_defaults<<<g, 256, 0, st>>>(nv, status, lane, cursor, wait, ins, arr, s, v);
  for (int q = 0; q < n_parts && nv > 0; ++q) k_state_cold<<<g, 256, 0, st>>>(parts[q], nv, status, wait, ins, arr);
  for (int q = 0; q < n_parts; ++q)
    if (parts[q].n_own > 0)
      k_state_driving<<<(parts[q].n_own + 7) / 8, 256, 0, st>>>(parts[q], status, lane, cursor, wait, s, v);
}

void launch_lane_stats(const StepArgs &a, int32_t *lane_count, int32_t *lane_wait,
                       float *road_speed, float zone, void *stream) {
  if (a.n_own > 0)
    k_lane_stats<<<(a.n_own + 3) / 4, 128, 0, (cudaStream_t)stream>>>(a, lane_count, lane_wait, road_speed, zone);
}

void launch_reduce_groups(const long long *tacc, int n_tiles, const int32_t *tiles, int n_own,
                          const int32_t *tile_group, const int32_t *cnt, const int32_t *icnt,
                          int n_groups, long long *out, void *stream) {
  cudaMemsetAsync(out, 0, (size_t)n_groups * (kNAcc + 1) * sizeof(long long), (cudaStream_t)stream);
  k_reduce_groups<<<296, 256, 0, (cudaStream_t)stream>>>(tacc, n_tiles, tiles, n_own, tile_group, cnt,
                                                         icnt, out);
}

// set_vehicle_route: every DRIVING vehicle with patch[vid] >= 0
// restarts at cursor patch[vid] (0) of its new route; its cached next roads
// are refreshed in the slab or inbox record that holds it.
__global__ void k_patch_routes(StepArgs A, const int32_t *patch) {
  const int tile = A.tiles[blockIdx.x];
  const int ns = A.cnt_in[tile], ni = A.icnt_in[tile];
  InboxRec *rec = const_cast<InboxRec *>(tile_recs(A, tile, ns));
  for (int i = threadIdx.x; i < ns + ni; i += blockDim.x) {
    InboxRec *r = rec + i;
    const int vid = r->vid;
    uint32_t *meta = &r->meta;
    int32_t *nxt = &r->nxt, *nxt2 = &r->nxt2;
    const int c = patch[vid];
    if (c < 0) continue;
    const int off = A.route_start[vid], len = A.route_len[vid];
    *meta = (*meta & 0xffffu) | ((uint32_t)c << 16);
    *nxt = c + 1 < len ? A.route[off + c + 1] : -1;
    *nxt2 = c + 2 < len ? A.route[off + c + 2] : -1;
    r->end_s = A.end_s[vid];                        // the new destination's end position
  }
}

// set_vehicle_route support: where is each vehicle of a batch (want[vid] =
// batch index b)?  out[2b] = cursor, out[2b+1] = global lane (DRIVING only).
__global__ void k_locate(StepArgs A, const int32_t *want, int32_t *out) {
  const int tile = A.tiles[blockIdx.x];
  const int ns = A.cnt_in[tile], ni = A.icnt_in[tile];
  const int l0 = A.tile_lane_off[tile];
  const InboxRec *rec = tile_recs(A, tile, ns);
  for (int i = threadIdx.x; i < ns + ni; i += blockDim.x) {
    const int vid = rec[i].vid;
    const uint32_t meta = rec[i].meta;
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

