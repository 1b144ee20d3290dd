// dev.h — device data layout of the B200 simulation store.
//
// Vehicles live in road TILES: one tile = one road's lanes + the junction
// lanes leaving that road (their only predecessor is one of its lanes).  Every
// vehicle is owned by exactly one tile; lane changes and road-lane -> junction
// lane hand-offs stay inside the tile, only junction lane -> next road
// hand-offs (and direct road -> road links) cross tiles.
//
// Between steps the state of a tile is
//   * its STAYERS: a compacted SoA slab segment sorted by (lane_local, s, vid)
//     (the paper's per-lane linked lists, as memory order), and
//   * its INBOX: unsorted 32-byte records of vehicles that entered the tile or
//     changed lane during the last step (the paper's per-lane addition
//     buffers), merged into the order at the start of the next step.
#pragma once
#include <stdint.h>

#include <utility>

#include <cuda_runtime.h>

namespace sim {

constexpr int kMaxTileLanes = 32;    // lanes per tile (road lanes + outgoing junction lanes)
constexpr int kThreads = 32;         // k_step block size: one warp per road tile
#ifndef KSMEM_VEH
#define KSMEM_VEH 112
#endif
constexpr int kSmemVeh = KSMEM_VEH;  // snapshot slots held in shared memory (larger tiles use global scratch)
constexpr int kSmemInbox = 48;       // inbox keys sorted in shared memory
constexpr int kNAcc = 12;            // per-tile int64 accumulators
constexpr int kMaxRoadLanes = 8;     // lanes per road (validated; 8-bit lane masks)
constexpr int kMaxSucc = 8;          // successors per road lane cached in the table
// tile descriptor (int32 words, 16-B padded, host-built by build_desc and
// rebuilt after setters): [nl, nroad, ne, n_all], glob[nl], len[nl], vmax[nl],
// flags[nl] (bit0 usable; road lanes: usable successors << 8, groups << 16),
// xl[nl] (junction lanes: exit lane, road lanes -1), per road lane 6 words
// (gbeg[0..3] bytes, gbeg[4], gtroad[0..3]), zero words up to a multiple of 4
// (desc_ent_off), then the ne usable successors of the road lanes sorted by
// (lane, target road, lane id), 8 words (16-B aligned, the layout of
// SuccEnt) each: j, target road, exit lane, flags (bit0 junction lane, lane
// << 8, rank k << 16, tile-local index of j << 24), outroads(exit lane) x4,
// padded to n_all entries; then the target-road section (kDescTroadWords).
// k_step reads the successor entries and the target-road section in place in
// the tile's ring slot (tile_setup rewrites each entry's flags word there)
__host__ __device__ constexpr int desc_ent_off(int nl, int nroad) { return (4 + 5 * nl + 6 * nroad + 3) & ~3; }
constexpr int kMaxGroups = 4;        // distinct target roads per road lane in the table
// target-road section at the end of a descriptor: ntr, umask, troad[16],
// reach[16] (bytes), gidx[4][16] (bytes)
constexpr int kDescTroadWords = 2 + kMaxRoadLanes * kMaxGroups + (kMaxRoadLanes * kMaxGroups) / 4 +
                                (kMaxRoadLanes * kMaxRoadLanes * kMaxGroups) / 4;
constexpr int kDescMaxWords = 4 + 5 * kMaxTileLanes + 6 * kMaxRoadLanes + 3 + 8 * kMaxRoadLanes * kMaxSucc +
                              kDescTroadWords + 3;
constexpr int kSmemProf = 8;         // profiles staged in shared memory
constexpr uint64_t kEmptyKey = ~0ull;

enum Acc {
  ACC_VEH_STEPS = 0, ACC_FINISHED, ACC_SUM_TRAVEL, ACC_SUM_WAIT_FIN, ACC_SUM_DELAY,
  ACC_LANE_CHANGES, ACC_HANDOFFS, ACC_INSERTED, ACC_GUARD, ACC_OVERFLOW,
  ACC_SUM_INSERT,   // sum of insert_time added at insertion, subtracted at arrival (att_all)
  ACC_R2
};
enum { ST_PENDING = 0, ST_DRIVING = 1, ST_FINISHED = 2 };
enum { SIG_GREEN = 0, SIG_YELLOW = 1, SIG_RED = 2 };
enum { POL_NONE = 0, POL_FIXED = 1, POL_MANUAL = 2, POL_MAXP = 3 };
enum { KIND_NORMAL = 0, KIND_DYNAMIC = 1, KIND_TIDAL = 2 };
constexpr int kLaneDest = -2, kLaneBlocked = -3;

struct Prof {                       // one vehicle profile
  float a_max, a_comf, T, s0, vmax, len, inv2sqrt_f, pad;
  double a_max_d, a_comf_d, T_d, s0_d, vmax_d, len_d, inv2sqrt_d, pad_d;
};

static_assert(sizeof(Prof) % 16 == 0, "Prof is copied as int4 words");

struct __align__(16) InboxRec {      // 32 B vehicle record (stayer or inbox), one sector
  float s, v;
  int32_t vid, nxt, nxt2;
  uint32_t meta;                    // lane_local:8 | profile:8 | cursor:16
  int32_t wait;
  float end_s;                      // end position on the destination road (trip input, carried
};                                  // so the step needs no per-vehicle global read)

// Gathered by the producer warp of k_step for every junction lane of a tile
// (DESIGN §3.2): the first vehicle of the junction lane's exit lane at t (the
// lookahead target of P:168-169 one lane beyond the tile) and the signal of
// the junction lane at t.
struct ExtFirst {
  float s, v, len, Lb;              // position / speed / vehicle length; Lb = length of the exit lane
  int32_t vid;                      // -1: the exit lane is empty
  int32_t sig;                      // signal of the junction lane at t
  int32_t b;                        // the exit lane
  // where a vehicle handed off into b goes (its tile's inbox): tile, b's
  // tile-local index, the tile's inbox start and capacity, the owner partition
  int32_t dtile, dlocal, dibase, dicap, downer;
};
static_assert(sizeof(ExtFirst) == 48, "ExtFirst: 12 words (16-B multiple for bulk copies)");
constexpr int kExtWords = (int)(sizeof(ExtFirst) / 4);

// Head of a road lane's pending-departure queue at t (K11), gathered
// by the producer warp: k = vid (-1: none due), its depart step, start
// position and profile, h = queue position.
struct PendHead {
  int32_t k, depart, prof, h;
  float start_s;
  int32_t pad[3];
};

struct MigRec {                     // 48 B: a vehicle migrating to another partition
  InboxRec rec;                     // rec.meta holds the destination lane's tile-local index
  int32_t tile, insert_time, pad0, pad1;
};                                  // element 0 of every peer region is a header: rec.vid = count

struct HaloRec {                    // 16 B: first-vehicle summary of one lane for a peer
  unsigned long long key;
  float v;
  int32_t pad;
};


// Direct peer-memory transport: the device
// buffers of partition q that other partitions write into (movers entering
// q's tiles, first-vehicle summaries and lane counts of q's lanes) or read
// (q's summaries / counts at t), indexed by the step parity like Part's own.
// In one process (loopback) these are the partitions' own pointers; across
// processes they are CUDA IPC mappings (NVLink peer memory on a multi-GPU box).
struct PeerView {                   // pointers only (exported as an array of handles)
  InboxRec *inbox[2];               // vehicle records (stayers + inboxes, by step parity)
  int32_t *icnt[2];
  unsigned long long *summ[3];
  float *pubv[2];
  int32_t *lcnt[3];
  int32_t *insert_time;
  uint8_t *status;
  unsigned int *bar;                // barrier arrival counter of partition q
  int32_t *cnt[2];                  // stayer counts and pending-queue heads: moved when a
                                    // tile changes owner (sim_repartition)
  int32_t *pend_head;
  int32_t *arrive_time, *wait_fin;  // read by sim_read_state_global
  void *xbuf[4];                    // reduction buffers: counters, lane statistics, group metrics,
                                    // host-call exchange (set_vehicle_route: where each vehicle is)
};


__host__ __device__ inline uint32_t pack_meta(int lane_local, int prof, int cursor) {
  return (uint32_t)lane_local | ((uint32_t)prof << 8) | ((uint32_t)cursor << 16);
}

struct StepArgs {
  // the step t this launch computes (t -> t+1) is t + *t_base when t_base is
  // set (a step of a captured CUDA graph: t is the step's offset in the graph,
  // *t_base the graph's first step, written before every replay), else t
  int32_t t, n_tiles, n_lanes, n_veh;
  const int32_t *t_base;
  uint64_t seed;
  // model constants (fp32 inputs; fp64 copies are their exact promotions)
  float polite, b_hard, b_safe, v_wait;
  double start_margin;              // v_cap + 0.5 * a_cap (ledger L17)
  int32_t lookahead, exact_mode, record, n_prof;
  // lanes (global id)
  const float *lane_len, *lane_vmax;
  const int32_t *lane_road;         // -1 junction lane
  const int32_t *lane_left, *lane_right;
  const int32_t *succ_off, *succ;
  const int32_t *target_road;       // road reached through lane j
  const int32_t *exit_lane;         // junction lane: its successor; road lane: itself
  const uint8_t *usable;
  const int4 *outroads;             // per lane: <= 4 distinct roads reachable through usable
                                    // successors (-1 pad; <= 4 validated at create)
  const uint8_t *lane_sig;
  const int32_t *lane_tile;
  const uint8_t *lane_local;
  // tiles (n_tiles global; this partition processes tiles[0 .. n_own))
  int32_t rank, n_own;
  const int32_t *tiles, *tile_owner;  // tiles: own tiles, largest slot capacity first
  int32_t *work;                    // [2] persistent-kernel work counter + finished warps (zero between launches)
  // k_step_w's tile order, rebuilt by k_prep every step: own tiles bucketed
  // by an estimate of their work at t (vehicles + 4 x lanes),
  // largest first (kNBucket buckets of 2^kBucketShift); bucket d's tiles at
  // bk_list[d * n_tiles ...];
  // bk_cnt is zero between steps (k_step_w's last CTA clears it)
  int32_t *bk_cnt, *bk_list;
  const int32_t *tile_lane_off, *tile_lanes, *tile_nroad;
  int32_t *desc;                    // tile blocks: descriptor words, then the k_prep staging
  const int32_t *desc_off;          // (ExtFirst per junction lane, PendHead per road lane)
  const int32_t *tile_base, *tile_cap, *tile_ibase, *tile_icap;
  int32_t *cnt_in, *cnt_out;        // [n_tiles] stayer counts (read / write buffers)
  int32_t *icnt_in, *icnt_out;      // [n_tiles] inbox counts
  // vehicle records of t (in) and t+1 (out), 32 B each: tile T
  // owns [tile_base, tile_base + cap + icap); its stayers are right-aligned in
  // [tile_base + cap - cnt, tile_base + cap), sorted by (lane_local, s, vid),
  // its inbox follows at tile_ibase = tile_base + cap, so one contiguous copy
  // fetches both
  const InboxRec *vin;
  InboxRec *vout;
  uint32_t *scratch;                // snapshot of tiles in global mode, at 8 x tile_base words (stride cap + icap)
  int32_t *bsort_scratch;           // [slots] inbox sort order of tiles in global mode (at tile_ibase)
  // per tile, static (host-built): {base, ibase, cap, icap}, {block offset,
  // block words, lanes, road lanes}, {descriptor words (= where the k_prep
  // staging starts), 0, 0, 0}
  const int4 *tinfo;
  uint32_t *pscratch;               // pass state of tiles in global mode: 10 words per slot at
                                    // 10 x (tile_base + 4 x tile)
  // migration to other partitions (world > 1): per-peer regions of MigRec
  MigRec *out_buf;
  const int32_t *out_off, *out_cap;
  int32_t *out_cnt;
  // lane summaries (first vehicle key) for t, t+1, t+2 (triple buffer)
  const unsigned long long *summ_cur;
  unsigned long long *summ_next, *summ_clear;
  const float *pubv_cur;            // [n_veh] speed of summary vehicles at t
  float *pubv_next;
  // cold per-vehicle data
  const int32_t *route_start, *route_len, *route;   // per vehicle: its roads route[start .. start+len)
  const float *end_s;
  const uint8_t *veh_prof;
  int32_t *insert_time, *arrive_time, *wait_fin;
  uint8_t *status;
  const int32_t *depart;
  const float *start_s;
  // pending queues (per lane, sorted by (depart, vid))
  const int32_t *pend_off, *pend_vid;
  int32_t *pend_head;
  const Prof *prof;
  long long *tacc;                  // [n_tiles][kNAcc]
  int32_t *lane_cnt_next;           // [n_lanes] vehicles per lane at t+1 (MAX_PRESSURE; NULL if unused)
  const uint64_t *veh_seed;         // [n_veh] Philox key per vehicle (batched environments) or NULL
  const int32_t *rng_id;            // [n_veh] Philox counter id per vehicle or NULL (= vid)
  // decision recording (vid-indexed), optional
  const PeerView *peers;            // [world] direct transport (NEXT-2), else NULL
  int32_t *r_leader, *r_of, *r_side;
  int8_t *r_hops, *r_phantom, *r_lc, *r_hand, *r_fin, *r_ins;
  float *r_acc;
  uint8_t *r_guard, *r_mark;        // r_mark: processed by this partition in the last step
};

#ifdef __CUDACC__
__device__ __forceinline__ int step_t(const StepArgs &A) {
  return A.t_base ? A.t + __ldg(A.t_base) : A.t;
}
// Programmatic dependent launch (the step kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): wait until the previous
// kernel of the stream has completed and its writes are visible; then let the
// next one be scheduled.  Both are no-ops without a programmatic dependency.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif

// the vehicles of tile T at t, stayers (sorted) then inbox records, contiguous
__host__ __device__ inline const InboxRec *tile_recs(const StepArgs &A, int T, int n_st) {
  return A.vin + A.tile_base[T] + A.tile_cap[T] - n_st;
}

struct SignalArgs {
  int32_t n_junctions, yellow;
  uint8_t *policy;
  int32_t *phase, *elapsed, *yellow_left, *pending, *request;
  int32_t *pol_request;             // set_tl_policy requests (-1 none), applied before `request`
  int32_t *remaining;               // MANUAL set_tl_duration green steps left (-1 none, L43)
  int32_t *dur_request;             // set_tl_duration requests (-1 none), applied after `request`
  const int32_t *jl_off, *jl;       // junction -> lanes (slots)
  const int32_t *ph_off;            // junction -> phases
  const int64_t *green_off;         // junction -> first byte of its phase rows
  const uint8_t *green;
  const int32_t *green_steps;
  uint8_t *lane_sig;
  // MAX_PRESSURE: per junction-lane slot its predecessor
  // and successor lane, lane vehicle counts of state(t), decision period
  const int32_t *jl_pred, *jl_succ;
  const int32_t *lane_cnt;
  // direct transport: the count of lane x lives with its owner partition
  const PeerView *peers;            // NULL: lane_cnt holds every lane
  const int32_t *lane_tile, *tile_owner;
  int32_t cnt_buf;                  // index of the lcnt buffer of state(t)
  int32_t mp_period;
};

constexpr int kNBucket = 64, kBucketShift = 3;

// A kernel launch that may begin while the previous kernel of the stream is
// still running (programmatic dependent launch): the kernel
// calls pdl_wait() before it reads what that kernel wrote.
template <typename... K, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
#ifdef KS_NO_PDL
  cfg.numAttrs = 0;                                 // dev builds: plain stream order
#else
  cfg.numAttrs = 1;
#endif
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// kernel launchers (kernels.cu)
void launch_set_i32(int32_t *p, int32_t v, void *stream);
void launch_signal(const SignalArgs &a, void *stream);
void launch_step(const StepArgs &a, void *stream, int smem_bytes);
void init_step_launch(int smem_bytes);             // function attributes / occupancy, once
void launch_prep(const StepArgs &a, void *stream);
void launch_lane_order(const StepArgs &a, int32_t *out_vid, uint8_t *out_lane, void *stream);
int step_smem_bytes();
void launch_apply_requests(int32_t *request, const int32_t *junc, const int32_t *phase, int m,
                           void *stream);
void launch_reduce_acc(const long long *tacc, int n_tiles, const int32_t *cnt,
                       const int32_t *icnt, const uint8_t *status, int nv, long long *out,
                       void *stream);
void launch_state_device(const StepArgs *parts, int n_parts, int nv, uint8_t *status, int32_t *lane,
                         int32_t *cursor, int32_t *wait, int32_t *ins, int32_t *arr, float *s, float *v,
                         void *stream);
void launch_lane_stats(const StepArgs &a, int32_t *lane_count, int32_t *lane_wait,
                       float *road_speed, float queue_zone, void *stream);
void launch_fill_u64(unsigned long long *p, unsigned long long v, int64_t n, void *stream);
void launch_patch_routes(const StepArgs &a, const int32_t *patch, void *stream);
void launch_locate(const StepArgs &a, const int32_t *want, int32_t *out, void *stream);
void launch_scatter_i32(int32_t *dst, const int32_t *idx, const int32_t *val, int32_t cval, int m,
                        void *stream);
void launch_scatter_f32(float *dst, const int32_t *idx, const float *val, int m, void *stream);
void launch_gather_u8(const uint8_t *src, const int32_t *idx, uint8_t *out, int m, void *stream);
void launch_reduce_groups(const long long *tacc, int n_tiles, const int32_t *tiles, int n_own,
                          const int32_t *tile_group, const int32_t *cnt, const int32_t *icnt,
                          int n_groups, long long *out, void *stream);
void launch_mig_header(MigRec *out_buf, const int32_t *out_off, const int32_t *out_cap,
                       int32_t *out_cnt, int world, void *stream);
void launch_absorb(const StepArgs &a, const MigRec *in_buf, const int32_t *in_off,
                   const int32_t *in_cap, int world, void *stream);
void launch_barrier(const PeerView *peers, int world, int rank, unsigned target, int32_t *err,
                    unsigned long long timeout_ns, void *stream);
void launch_peer_sum(const PeerView *peers, int world, int kind, int dtype, int64_t off, int64_t n,
                     void *out, void *stream);
void launch_rehome(const StepArgs &a, const int32_t *new_owner, void *stream);
void launch_tile_counts(const StepArgs &a, int32_t *out, void *stream);
void launch_halo_pack(const StepArgs &a, const int32_t *lanes, HaloRec *buf, int64_t n, void *stream);
void launch_halo_unpack(const StepArgs &a, const int32_t *lanes, const HaloRec *buf, int64_t n,
                        void *stream);

}  // namespace sim
