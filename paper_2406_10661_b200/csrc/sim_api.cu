// sim_api.cu — host runtime behind include/sim.h.
//
// Builds road tiles (dev.h), validates inputs, partitions the
// tiles over ranks, owns all device memory, uploads canonical
// (per-lane sorted) state, enqueues steps (k_signal + k_step per partition,
// then the migration and halo exchanges when partitioned) on the handle's
// stream, and implements the setters / readers.  Nothing here computes the
// model: every per-vehicle decision is taken on the GPU (kernels.cu, model.cuh).
//
// Partitioned modes (sim_params.world > 1):
//   * NCCL: one process per GPU, one partition per handle; exchanges are
//     grouped ncclSend / ncclRecv on the simulation stream; metrics are
//     ncclAllReduce'd (NCCL is loaded with dlopen only in this mode);
//   * loopback: all `world` partitions live in one handle on one device and
//     exchange by device-to-device copies — the same kernels and exchange
//     plan, used to test partition invariance (P-PART) on a single GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/sim.h"
#include "dev.h"

using namespace sim;

namespace {
thread_local std::string g_create_err;
std::mutex g_live_mu;
std::set<const void *> g_live;      // live handles: calls on destroyed handles fail
bool is_live(const void *h) {
  std::lock_guard<std::mutex> lk(g_live_mu);
  return g_live.count(h) != 0;
}

struct HostState {                  // vid / junction / lane indexed state
  int t = 0;
  std::vector<uint8_t> status;
  std::vector<int> lane, cursor, wait, insert_time, arrive_time;
  std::vector<float> s, v;
  std::vector<uint8_t> jpol;
  std::vector<int> jphase, jel, jy, jpend, jrem;
  std::vector<uint8_t> dir;
  std::vector<uint8_t> to_inbox;     // test hook: 1 = place this DRIVING vehicle in its tile's inbox
};

// ---- minimal NCCL binding (dlopen; only the partitioned NCCL mode needs it) --
typedef struct { char internal[128]; } NcclId;
typedef void *NcclComm;
struct Nccl {
  void *lib = nullptr;
  int (*GetUniqueId)(NcclId *) = nullptr;
  int (*CommInitRank)(NcclComm *, int, NcclId, int) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  int (*Send)(const void *, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*Recv)(void *, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*AllReduce)(const void *, void *, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(int) = nullptr;
  bool load(std::string &err) {
    if (lib) return true;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names)
      if ((lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!lib) { err = "cannot dlopen libnccl.so.2 (needed for world > 1 without loopback)"; return false; }
#define SYM(f, n) f = reinterpret_cast<decltype(f)>(dlsym(lib, n)); if (!f) { err = std::string("missing ") + n; return false; }
    SYM(GetUniqueId, "ncclGetUniqueId"); SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy"); SYM(Send, "ncclSend"); SYM(Recv, "ncclRecv");
    SYM(AllReduce, "ncclAllReduce"); SYM(GroupStart, "ncclGroupStart"); SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    return true;
  }
};
Nccl g_nccl;
constexpr int kNcclInt8 = 0, kNcclInt64 = 4, kNcclSum = 0;
}  // namespace

// One partition's device state (all partitions of a loopback handle share the
// device and the stream; a NCCL handle has exactly one).
struct Part {
  int rank = 0;
  StepArgs A{};
  SignalArgs SG{};
  InboxRec *inbox[2]{};
  int32_t *cnt[2]{}, *icnt[2]{};
  unsigned long long *summ[3]{};
  float *pubv[2]{};
  int32_t *pend_off_d = nullptr, *pend_vid_d = nullptr, *pend_head_d = nullptr;
  uint8_t *usable_d = nullptr;
  int32_t *outroads_d = nullptr;
  int32_t *desc_d = nullptr;
  long long *red_d = nullptr;
  int32_t *lanestat_d = nullptr;
  int32_t *tile_group_d = nullptr;              // batched environments: group of each tile
  float *lane_vmax_d = nullptr;                 // writable alias of A.lane_vmax (set_lane_max_speed)
  int32_t *route_start_d = nullptr, *route_len_d = nullptr, *route_d = nullptr;   // writable aliases
  float *end_s_d = nullptr;
  int32_t *patch_d = nullptr;                   // [n_veh] set_vehicle_route: new cursor or -1
  long long *grp_d = nullptr;                   // [n_groups][kNAcc + 1]
  std::vector<int> tiles;                       // own tiles
  // exchange plan (world > 1): migrant regions per peer (header record + cap)
  std::vector<int> out_off, out_cap, in_off, in_cap;
  MigRec *out_buf = nullptr, *in_buf = nullptr;
  int32_t *out_cnt = nullptr;
  int32_t *in_off_d = nullptr, *in_cap_d = nullptr;
  int64_t out_n = 0, in_n = 0;
  // halo: summaries of lanes each peer reads from us / we read from each peer
  std::vector<int> hs_off, hr_off;              // [world+1] offsets into the lists
  int32_t *hs_lanes = nullptr, *hr_lanes = nullptr;
  HaloRec *hs_buf = nullptr, *hr_buf = nullptr;
  int64_t hs_n = 0, hr_n = 0;
  // direct transport (NEXT-2): this partition's exported buffers and the
  // device table of every partition's buffers
  PeerView view{};
  unsigned int *bar_d = nullptr;
  PeerView *peers_d = nullptr;
  int32_t *tiles_cap_d = nullptr;               // sim_repartition: own-tile list (capacity n_tiles)
  int32_t *xch_d = nullptr;                     // multi-process: host-call exchange, 3 x n_veh
  int32_t *lo_vid_d = nullptr;                  // sim_read_state lane order (k_lane_order), n_slots
  uint8_t *lo_lane_d = nullptr;
};

struct sim_s {
  std::string err;
  sim_status sticky = SIM_OK;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // graph (host copies)
  int nl = 0, nr = 0, nj = 0, nv = 0, nt = 0;
  std::vector<float> L, vmax;
  std::vector<int> road, junc, left, right, succ_off, succ, pred, target_road, exit_lane;
  std::vector<uint8_t> kind, turn;
  std::vector<int> partner;
  std::vector<int> road_off, road_lanes, jl_off, jl, ph_off, green_steps;
  std::vector<int64_t> green_off;
  std::vector<uint8_t> green, pol0;
  std::vector<int> offset0;
  // tiles
  std::vector<int> tile_lane_off, tile_lanes, tile_nroad, tile_base, tile_cap, tile_ibase, tile_icap;
  std::vector<int> lane_tile;
  std::vector<uint8_t> lane_local;
  int64_t n_slots = 0;                          // vehicle record slots (all tiles' regions)
  // trips
  std::vector<int> route_off, route, depart, start_lane;
  std::vector<int> rstart, rlen;                // per vehicle: route[rstart .. rstart + rlen) (set_vehicle_route appends)
  std::vector<std::vector<int>> radj;           // road -> roads reachable through one lane connection
  int64_t route_cap = 0;                        // device route buffer capacity (entries)
  std::vector<float> start_s, start_v, end_s;
  std::vector<uint8_t> vprof, on0;
  // params
  sim_params P{};
  std::vector<Prof> profs;
  double start_margin = 0;
  int Y = 3;
  // partitioning
  int world = 1, rank = 0;                      // rank: this process (NCCL mode)
  bool loopback = false;
  bool direct = false;                          // NEXT-2: k_step writes into the owner's buffers
  bool ipc = false;                             // direct across processes (CUDA IPC mappings)
  bool connected = false;                       // ipc: sim_ipc_connect done
  unsigned bar_epoch = 0;                       // ipc: barriers passed
  unsigned long long bar_timeout_ns = 60000000000ull;  // ipc: params.barrier_timeout_ms (default 60 s)
  int32_t *bar_err_d = nullptr;                 // ipc: set by a barrier that timed out
  void *ipc_tmp = nullptr;                      // ipc: reduction result buffer
  std::vector<void *> ipc_opened;               // ipc: peer mappings to close
  int32_t *repart_own_d = nullptr;              // sim_repartition: new owners (device)
  std::vector<PeerView> peer_views;             // ipc: every rank's buffers (host copy of the table)
  std::vector<int> tile_owner;
  NcclComm comm = nullptr;
  std::vector<Part> parts;
  // state
  int t = 0;
  std::vector<uint8_t> dir, usable;
  std::vector<int32_t> outroads;     // [4 * n_lanes]
  std::vector<int32_t> desc, desc_off;   // tile blocks: descriptor (dev.h) + k_prep staging
  std::vector<int32_t> desc_words;       // per tile: words of the descriptor part
  int64_t fin0 = 0;                  // FINISHED vehicles in the last loaded state
  long long acc_fin0 = 0;            // finished counter at the last load
  int64_t ins0 = 0;                  // sum of insert_time over the DRIVING vehicles loaded
  long long acc_ins0 = 0;            // ACC_SUM_INSERT at the last load
  // batched environments (NEXT-3)
  std::vector<uint64_t> vseed;
  std::vector<int32_t> rngid, road_group, veh_group;
  int n_groups = 0;
  std::vector<long long> grp_nv, grp_fin0, grp_acc_fin0;
  // device
  std::vector<void *> allocs;
  std::vector<uint8_t> alloc_hooked;            // 1: allocs[i] came from params.alloc
  int64_t bytes = 0;
  int32_t *stage_d = nullptr;        // device staging for batch setters
  int stage_cap = 0;
  uint8_t *stage_dir_d = nullptr;    // device staging for lane-direction setters
  void *pinned = nullptr;
  size_t pinned_cap = 0;
  std::vector<int> req_mark;                    // set_signal_phase_batch: last entry per junction
  std::vector<uint8_t> restricted;              // set_lane_restriction flags (L44)
  int32_t *lcnt[3] = {nullptr, nullptr, nullptr}; // MAX_PRESSURE lane counts for t, t+1, t+2 (mod 3)
  bool any_maxp = false;                        // some junction runs MAX_PRESSURE
  std::vector<int> jl_pred, jl_succ;            // per junction-lane slot: predecessor / successor lane
  int req_epoch = 0;
  void *rd_pinned = nullptr;                    // read_metrics: counters + lane statistics
  size_t rd_cap = 0;
  cudaEvent_t stage_ev = nullptr;
  int smem = 0;
  // device timing windows (sim_enable_timing / sim_read_timing)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  int64_t n_launch = 0;
  // sim_step(n) as replays of a captured CUDA graph of kGraphSteps steps
  // (DESIGN §3.2): the graph's kernels read the absolute step from t_dev
  int32_t *t_dev = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::vector<unsigned char> g_fp;              // host state the graph was captured from
  int64_t g_launches = 0;                       // kernels per replay
  bool g_off = false;                           // capture unavailable on this stream
};

namespace {

sim_status fail(sim_s *h, sim_status st, const std::string &m) {
  if (h) h->err = m; else g_create_err = m;
  return st;
}

#define CK(h, x)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      (h)->sticky = SIM_E_CUDA;                                                     \
      return fail((h), SIM_E_CUDA, std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                       " at " + #x);                                \
    }                                                                               \
  } while (0)

#define NK(h, x)                                                                    \
  do {                                                                              \
    int r_ = (x);                                                                   \
    if (r_ != 0) {                                                                  \
      (h)->sticky = SIM_E_NCCL;                                                     \
      return fail((h), SIM_E_NCCL, std::string("NCCL: ") + g_nccl.GetErrorString(r_) + \
                                       " at " + #x);                                \
    }                                                                               \
  } while (0)

// cudaMemset on the handle's stream, completed before returning: the legacy
// default stream is not ordered with a non-blocking handle stream, so a plain
// cudaMemset could land after (or before) the stream work that follows it
cudaError_t dmemset(sim_s *h, void *p, int v, size_t bytes) {
  cudaError_t e = cudaMemsetAsync(p, v, bytes, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  return e;
}

template <typename T>
sim_status dalloc(sim_s *h, T **p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  if (h->P.alloc) {                                 // caller's allocator (e.g. PyTorch's caching one)
    *p = reinterpret_cast<T *>(h->P.alloc(n * sizeof(T), h->P.alloc_ctx));
    if (!*p) return fail(h, SIM_E_OOM, "params.alloc returned NULL");
  } else {
    cudaError_t e = cudaMalloc((void **)p, n * sizeof(T));
    if (e != cudaSuccess) {
      return fail(h, SIM_E_OOM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    }
  }
  h->allocs.push_back(*p);
  h->alloc_hooked.push_back(h->P.alloc ? 1 : 0);
  // zero-filled: unused slots of the record regions are read whole by the
  // state reads (compute-sanitizer initcheck clean).  On the handle's stream
  // and completed here: a cudaMemset on the legacy default stream is not
  // ordered with a non-blocking handle stream, so a buffer allocated lazily
  // (the lane-order buffers of sim_read_state, the step-graph t word) could
  // be zeroed after the kernel that filled it had run
  cudaError_t ez = cudaMemsetAsync(*p, 0, n * sizeof(T), h->stream);
  if (ez == cudaSuccess) ez = cudaStreamSynchronize(h->stream);
  if (ez != cudaSuccess) return fail(h, SIM_E_CUDA, std::string("cudaMemset: ") + cudaGetErrorString(ez));
  h->bytes += (int64_t)(n * sizeof(T));
  return SIM_OK;
}

template <typename T>
sim_status upload(sim_s *h, T **p, const std::vector<T> &v) {
  sim_status st = dalloc(h, p, v.size());
  if (st) return st;
  if (!v.empty()) CK(h, cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return SIM_OK;
}

bool is_road(const sim_s *h, int l) { return h->road[l] >= 0; }

// Tile descriptors (layout in dev.h): static graph data + the usable flags /
// reachable roads that setters change; rebuilt by compute_usable.
void build_desc(sim_s *h) {
  if (h->tile_lane_off.empty()) return;
  h->desc.clear();
  h->desc_off.assign(h->nt + 1, 0);
  h->desc_words.assign(h->nt, 0);
  for (int T = 0; T < h->nt; ++T) {
    const int l0 = h->tile_lane_off[T], nl = h->tile_lane_off[T + 1] - l0, nroad = h->tile_nroad[T];
    // successor table of the road lanes (static between setters, so sorted and
    // grouped here): usable successors sorted by (target road, lane id), grouped
    // by target road; per road lane 6 words: gbeg[0..4] as bytes, gtroad[0..3]
    std::vector<int32_t> ent, grp;
    std::vector<int32_t> lane_sn(nroad, 0), lane_ng(nroad, 0);
    int n_all = 0;                                  // all successors: fixes the descriptor size
    for (int l = 0; l < nroad; ++l) {
      const int g = h->tile_lanes[l0 + l];
      n_all += h->succ_off[g + 1] - h->succ_off[g];
      std::vector<int> js;
      for (int e = h->succ_off[g]; e < h->succ_off[g + 1]; ++e)
        if (h->usable[h->succ[e]]) js.push_back(h->succ[e]);
      std::sort(js.begin(), js.end(), [&](int a, int b) {
        return h->target_road[a] != h->target_road[b] ? h->target_road[a] < h->target_road[b] : a < b;
      });
      uint8_t gbeg[kMaxGroups + 1] = {0, 0, 0, 0, 0};
      int32_t gtr[kMaxGroups] = {-1, -1, -1, -1};
      int ng = 0;
      for (int k = 0; k < (int)js.size(); ++k) {
        const int j = js[k], b = h->exit_lane[j];
        if (k == 0 || h->target_road[js[k - 1]] != h->target_road[j]) {
          if (ng < kMaxGroups) { gbeg[ng] = (uint8_t)k; gtr[ng] = h->target_road[j]; }
          ++ng;
        }
        ent.push_back(j);
        ent.push_back(h->target_road[j]);
        ent.push_back(b);
        // bits 24-31: tile-local index of j when j is a junction lane (it then
        // belongs to this tile), 0xff for a direct road -> road link
        const uint32_t jl = is_road(h, j) ? 0xffu : (uint32_t)h->lane_local[j];
        ent.push_back((int32_t)((is_road(h, j) ? 0u : 1u) | ((uint32_t)l << 8) | ((uint32_t)k << 16) | (jl << 24)));
        for (int q = 0; q < 4; ++q) ent.push_back(h->outroads[4 * (size_t)b + q]);
      }
      if (ng <= kMaxGroups) gbeg[ng] = (uint8_t)js.size();
      lane_sn[l] = (int)js.size();
      lane_ng[l] = ng;
      grp.push_back((int32_t)(gbeg[0] | (gbeg[1] << 8) | (gbeg[2] << 16) | ((uint32_t)gbeg[3] << 24)));
      grp.push_back(gbeg[4]);
      for (int q = 0; q < kMaxGroups; ++q) grp.push_back(gtr[q]);
    }
    std::vector<int32_t> w{nl, nroad, (int)(ent.size() / 8), n_all};
    for (int l = 0; l < nl; ++l) w.push_back(h->tile_lanes[l0 + l]);
    for (int l = 0; l < nl; ++l) { float x = h->L[h->tile_lanes[l0 + l]]; int32_t b; std::memcpy(&b, &x, 4); w.push_back(b); }
    for (int l = 0; l < nl; ++l) { float x = h->vmax[h->tile_lanes[l0 + l]]; int32_t b; std::memcpy(&b, &x, 4); w.push_back(b); }
    for (int l = 0; l < nl; ++l)
      w.push_back((h->usable[h->tile_lanes[l0 + l]] ? 1 : 0) |
                  (l < nroad ? (lane_sn[l] << 8) | (lane_ng[l] << 16) : 0));
    // junction lanes: their exit lane (the producer warp of k_step gathers its
    // first vehicle at t); road lanes: -1
    for (int l = 0; l < nl; ++l) w.push_back(l < nroad ? -1 : h->exit_lane[h->tile_lanes[l0 + l]]);
    w.insert(w.end(), grp.begin(), grp.end());
    w.resize(desc_ent_off(nl, nroad), 0);            // 16-B aligned entries (read in place)
    w.insert(w.end(), ent.begin(), ent.end());
    // pad to all successors so setters (which change the usable set) never
    // change the descriptor's size or offsets
    w.insert(w.end(), (size_t)(n_all - (int)(ent.size() / 8)) * 8, 0);
    // target-road section (kDescTroadWords): the distinct roads the
    // road lanes lead to, numbered in order of first appearance over (lane,
    // group); reach[k] = road lanes with a group toward troad[k]; gidx[a][k] =
    // that group of lane a (-1 none); umask = usable road lanes
    {
      int32_t tw[kDescTroadWords] = {0};
      int ntr = 0;
      int troad[kMaxRoadLanes * kMaxGroups];
      uint8_t reach[kMaxRoadLanes * kMaxGroups] = {0};
      int8_t gidx[kMaxRoadLanes][kMaxRoadLanes * kMaxGroups];
      std::memset(gidx, 0xff, sizeof(gidx));
      uint32_t umask = 0;
      for (int a = 0; a < nroad; ++a) {
        if (h->usable[h->tile_lanes[l0 + a]]) umask |= 1u << a;
        const int32_t *gr = &grp[6 * (size_t)a];
        for (int g = 0; g < lane_ng[a] && g < kMaxGroups; ++g) {
          const int R = gr[2 + g];
          int k = 0;
          while (k < ntr && troad[k] != R) ++k;
          if (k == ntr) troad[ntr++] = R;
          reach[k] |= (uint8_t)(1u << a);
          gidx[a][k] = (int8_t)g;
        }
      }
      tw[0] = ntr;
      tw[1] = (int32_t)umask;
      for (int k = 0; k < kMaxRoadLanes * kMaxGroups; ++k) tw[2 + k] = k < ntr ? troad[k] : -1;
      std::memcpy(&tw[2 + kMaxRoadLanes * kMaxGroups], reach, sizeof(reach));
      std::memcpy(&tw[2 + kMaxRoadLanes * kMaxGroups + sizeof(reach) / 4], gidx, sizeof(gidx));
      w.insert(w.end(), tw, tw + kDescTroadWords);
    }
    while (w.size() % 4) w.push_back(0);
    // then room for what k_prep stages per step: an ExtFirst per
    // junction lane and a PendHead per road lane, so that the tile's whole
    // block is one bulk copy
    h->desc_words[T] = (int)w.size();
    w.insert(w.end(), (size_t)kExtWords * (nl - nroad) + (size_t)8 * nroad, 0);
    h->desc.insert(h->desc.end(), w.begin(), w.end());
    h->desc_off[T + 1] = (int)h->desc.size();
  }
}

// usable(ℓ) (ledger L29, L30)
void compute_usable(sim_s *h) {
  h->usable.assign(h->nl, 1);
  if (h->restricted.size() != (size_t)h->nl) h->restricted.assign(h->nl, 0);
  for (int l = 0; l < h->nl; ++l)
    if (is_road(h, l)) h->usable[l] = !h->restricted[l] && !(h->kind[l] == KIND_TIDAL && h->dir[l] != 0);
  for (int l = 0; l < h->nl; ++l) {
    if (is_road(h, l)) continue;
    int a = h->pred[l], b = h->succ[h->succ_off[l]];
    bool u = h->usable[b];
    if (u && h->kind[a] == KIND_DYNAMIC) {
      if (h->turn[l] == 1) u = h->dir[a] == 1;
      else if (h->turn[l] == 0) u = h->dir[a] == 0;
    }
    h->usable[l] = u && !h->restricted[l];
  }
  // outroads: distinct roads reachable through usable successors (<= 4, else -2 marker)
  h->outroads.assign(4 * (size_t)h->nl, -1);
  for (int l = 0; l < h->nl; ++l) {
    int k = 0;
    int32_t *o = &h->outroads[4 * (size_t)l];
    for (int e = h->succ_off[l]; e < h->succ_off[l + 1]; ++e) {
      int j = h->succ[e];
      if (!h->usable[j]) continue;
      int r = h->target_road[j];
      bool seen = false;
      for (int q = 0; q < k && q < 4; ++q) seen |= o[q] == r;
      if (seen) continue;
      if (k < 4) o[k] = r;
      ++k;
    }
  }
  build_desc(h);
}

sim_status validate_and_copy(sim_s *h, const sim_graph *g, const sim_trips *tr,
                             const sim_params *p) {
  if (!g || !tr || !p) return fail(h, SIM_E_INVALID, "null argument");
  if (p->dt != 1.0f) return fail(h, SIM_E_INVALID, "params.dt must be 1.0 (P:768)");
  if (p->n_profiles <= 0 || p->n_profiles > 256 || !p->profiles)
    return fail(h, SIM_E_INVALID, "n_profiles must be in [1, 256]");
  for (int i = 0; i < p->n_profiles; ++i) {
    const sim_profile &q = p->profiles[i];
    if (!(q.a_max > 0 && q.a_comf > 0 && q.T > 0 && q.s0 > 0 && q.v_max > 0 && q.length > 0))
      return fail(h, SIM_E_INVALID, "profile " + std::to_string(i) + " has a non-positive field");
  }
  if (p->lookahead_lanes < 0 || p->yellow_steps < 0)
    return fail(h, SIM_E_INVALID, "lookahead_lanes / yellow_steps must be >= 0");
  const int nl = g->n_lanes, nr = g->n_roads, nj = g->n_junctions, nv = tr->n_trips;
  if (nl <= 0 || nr <= 0 || nj < 0 || nv < 0) return fail(h, SIM_E_INVALID, "bad sizes");
  h->nl = nl; h->nr = nr; h->nj = nj; h->nv = nv;
  h->L.assign(g->lane_length, g->lane_length + nl);
  h->vmax.assign(g->lane_max_speed, g->lane_max_speed + nl);
  h->road.assign(g->lane_road, g->lane_road + nl);
  h->junc.assign(g->lane_junction, g->lane_junction + nl);
  h->left.assign(g->lane_left, g->lane_left + nl);
  h->right.assign(g->lane_right, g->lane_right + nl);
  h->succ_off.assign(g->succ_offsets, g->succ_offsets + nl + 1);
  h->kind.assign(g->lane_kind, g->lane_kind + nl);
  h->turn.assign(g->lane_turn, g->lane_turn + nl);
  h->partner.assign(g->tidal_partner, g->tidal_partner + nl);
  h->dir.assign(g->lane_dir0, g->lane_dir0 + nl);
  if (h->succ_off[0] != 0) return fail(h, SIM_E_INVALID, "succ_offsets[0] != 0");
  for (int l = 0; l < nl; ++l)
    if (h->succ_off[l + 1] < h->succ_off[l]) return fail(h, SIM_E_INVALID, "succ_offsets not monotone");
  h->succ.assign(g->succ_lanes, g->succ_lanes + h->succ_off[nl]);
  for (int l = 0; l < nl; ++l) {
    std::string id = " (lane " + std::to_string(l) + ")";
    if (!(h->L[l] > 0 && std::isfinite(h->L[l]))) return fail(h, SIM_E_INVALID, "lane_length must be > 0" + id);
    if (!(h->vmax[l] > 0 && std::isfinite(h->vmax[l]))) return fail(h, SIM_E_INVALID, "lane_max_speed must be > 0" + id);
    if ((h->road[l] >= 0) == (h->junc[l] >= 0)) return fail(h, SIM_E_INVALID, "lane must belong to exactly one road or junction" + id);
    if (h->road[l] >= nr || h->junc[l] >= nj) return fail(h, SIM_E_INVALID, "road/junction id out of range" + id);
    if (h->kind[l] > 2) return fail(h, SIM_E_INVALID, "bad lane_kind" + id);
    for (int e = h->succ_off[l]; e < h->succ_off[l + 1]; ++e)
      if (h->succ[e] < 0 || h->succ[e] >= nl) return fail(h, SIM_E_INVALID, "successor out of range" + id);
  }
  std::vector<std::vector<int>> preds(nl);
  for (int l = 0; l < nl; ++l)
    for (int e = h->succ_off[l]; e < h->succ_off[l + 1]; ++e) preds[h->succ[e]].push_back(l);
  h->pred.assign(nl, -1);
  h->target_road.assign(nl, -1);
  h->exit_lane.assign(nl, -1);
  for (int l = 0; l < nl; ++l) {
    std::string id = " (lane " + std::to_string(l) + ")";
    if (!is_road(h, l)) {
      if (h->succ_off[l + 1] - h->succ_off[l] != 1 || preds[l].size() != 1)
        return fail(h, SIM_E_INVALID, "junction lane needs exactly one predecessor and one successor" + id);
      int b = h->succ[h->succ_off[l]], a = preds[l][0];
      if (!is_road(h, b) || !is_road(h, a))
        return fail(h, SIM_E_INVALID, "junction lane must connect two road lanes" + id);
      if (h->left[l] >= 0 || h->right[l] >= 0)
        return fail(h, SIM_E_INVALID, "junction lanes have no left/right neighbours (P:95)" + id);
      h->pred[l] = a;
      h->target_road[l] = h->road[b];
      h->exit_lane[l] = b;
    } else {
      h->target_road[l] = h->road[l];
      h->exit_lane[l] = l;
    }
  }
  h->road_off.assign(g->road_lane_offsets, g->road_lane_offsets + nr + 1);
  if (h->road_off[0] != 0 || h->road_off[nr] < 0) return fail(h, SIM_E_INVALID, "bad road_lane_offsets");
  h->road_lanes.assign(g->road_lanes, g->road_lanes + h->road_off[nr]);
  std::vector<int> seen(nl, 0);
  for (int r = 0; r < nr; ++r) {
    std::string id = " (road " + std::to_string(r) + ")";
    int a = h->road_off[r], b = h->road_off[r + 1];
    if (b <= a) return fail(h, SIM_E_INVALID, "road without lanes" + id);
    for (int e = a; e < b; ++e) {
      int l = h->road_lanes[e];
      if (l < 0 || l >= nl || h->road[l] != r) return fail(h, SIM_E_INVALID, "road_lanes inconsistent with lane_road" + id);
      seen[l]++;
      if (h->L[l] != h->L[h->road_lanes[a]]) return fail(h, SIM_E_INVALID, "lanes of a road must have equal length (L20)" + id);
      int lf = e > a ? h->road_lanes[e - 1] : -1, rt = e + 1 < b ? h->road_lanes[e + 1] : -1;
      if (h->left[l] != lf || h->right[l] != rt)
        return fail(h, SIM_E_INVALID, "lane_left/lane_right must follow road_lanes order (leftmost first)" + id);
    }
  }
  for (int l = 0; l < nl; ++l)
    if (is_road(h, l) && seen[l] != 1) return fail(h, SIM_E_INVALID, "road lane missing from road_lanes");
  for (int l = 0; l < nl; ++l)
    if (h->kind[l] == KIND_TIDAL) {
      int q = h->partner[l];
      if (q >= 0 && (q >= nl || h->partner[q] != l || h->kind[q] != KIND_TIDAL))
        return fail(h, SIM_E_INVALID, "tidal_partner must be mutual (lane " + std::to_string(l) + ")");
    }
  // junctions
  h->jl_off.assign(g->junc_lane_offsets, g->junc_lane_offsets + nj + 1);
  h->jl.assign(g->junc_lanes, g->junc_lanes + (nj ? h->jl_off[nj] : 0));
  h->ph_off.assign(g->junc_phase_offsets, g->junc_phase_offsets + nj + 1);
  int nph = nj ? h->ph_off[nj] : 0;
  h->green_steps.assign(g->phase_green_steps, g->phase_green_steps + nph);
  h->pol0.assign(g->junc_policy, g->junc_policy + nj);
  h->offset0.assign(g->junc_offset_steps, g->junc_offset_steps + nj);
  h->green_off.assign(nj + 1, 0);
  h->jl_pred.assign(h->jl.size(), 0);
  h->jl_succ.assign(h->jl.size(), 0);
  for (size_t e = 0; e < h->jl.size(); ++e) {       // junction lanes: one predecessor, one successor
    const int l = h->jl[e];
    if (l >= 0 && l < nl) { h->jl_pred[e] = std::max(h->pred[l], 0); h->jl_succ[e] = h->succ[h->succ_off[l]]; }
  }
  for (int j = 0; j < nj; ++j) {
    int ns = h->jl_off[j + 1] - h->jl_off[j], np = h->ph_off[j + 1] - h->ph_off[j];
    if (ns < 0 || np < 0) return fail(h, SIM_E_INVALID, "bad junction CSR");
    for (int e = h->jl_off[j]; e < h->jl_off[j + 1]; ++e)
      if (h->jl[e] < 0 || h->jl[e] >= nl || h->junc[h->jl[e]] != j)
        return fail(h, SIM_E_INVALID, "junc_lanes inconsistent with lane_junction (junction " + std::to_string(j) + ")");
    if (h->pol0[j] > 3) return fail(h, SIM_E_INVALID, "bad junc_policy");
    for (int k = h->ph_off[j]; k < h->ph_off[j + 1]; ++k)
      if (h->pol0[j] == POL_FIXED && h->green_steps[k] < 1)
        return fail(h, SIM_E_INVALID, "FIXED_TIME green durations must be >= 1");
    h->green_off[j + 1] = h->green_off[j] + (int64_t)ns * np;
  }
  h->green.assign(g->phase_green, g->phase_green + h->green_off[nj]);
  // trips
  h->route_off.assign(tr->route_offsets, tr->route_offsets + nv + 1);
  if (h->route_off[0] != 0) return fail(h, SIM_E_INVALID, "route_offsets[0] != 0");
  h->route.assign(tr->route_roads, tr->route_roads + h->route_off[nv]);
  h->depart.assign(tr->depart_step, tr->depart_step + nv);
  h->start_lane.assign(tr->start_lane, tr->start_lane + nv);
  h->start_s.assign(tr->start_s, tr->start_s + nv);
  h->start_v.assign(tr->start_v, tr->start_v + nv);
  h->end_s.assign(tr->end_s, tr->end_s + nv);
  h->vprof.assign(tr->profile, tr->profile + nv);
  h->on0.assign(tr->on_network_at_t0, tr->on_network_at_t0 + nv);
  // road adjacency for route validation
  std::vector<std::vector<int>> radj(nr);
  for (int l = 0; l < nl; ++l)
    if (is_road(h, l))
      for (int e = h->succ_off[l]; e < h->succ_off[l + 1]; ++e) radj[h->road[l]].push_back(h->target_road[h->succ[e]]);
  for (auto &v : radj) { std::sort(v.begin(), v.end()); v.erase(std::unique(v.begin(), v.end()), v.end()); }
  for (int k = 0; k < nv; ++k) {
    std::string id = " (trip " + std::to_string(k) + ")";
    int a = h->route_off[k], b = h->route_off[k + 1];
    if (b <= a || b - a > 65000) return fail(h, SIM_E_INVALID, "route length must be in [1, 65000]" + id);
    for (int e = a; e < b; ++e) {
      int r = h->route[e];
      if (r < 0 || r >= nr) return fail(h, SIM_E_INVALID, "route road out of range" + id);
      if (e + 1 < b && !std::binary_search(radj[r].begin(), radj[r].end(), h->route[e + 1]))
        return fail(h, SIM_E_INVALID, "consecutive route roads are not connected" + id);
    }
    int sl = h->start_lane[k];
    if (sl < 0 || sl >= nl || h->road[sl] != h->route[a]) return fail(h, SIM_E_INVALID, "start_lane must be a lane of route[0]" + id);
    if (!(h->start_s[k] >= 0 && h->start_s[k] <= h->L[sl])) return fail(h, SIM_E_INVALID, "start_s outside [0, L]" + id);
    if (h->start_s[k] == 0.0f) h->start_s[k] = 0.0f;          // canonical +0
    if (!(h->start_v[k] >= 0 && std::isfinite(h->start_v[k]))) return fail(h, SIM_E_INVALID, "start_v must be >= 0" + id);
    int dl = h->road_lanes[h->road_off[h->route[b - 1]]];
    if (!(h->end_s[k] >= 0 && h->end_s[k] <= h->L[dl])) return fail(h, SIM_E_INVALID, "end_s outside [0, L]" + id);
    if (h->vprof[k] >= p->n_profiles) return fail(h, SIM_E_INVALID, "profile index out of range" + id);
    if (h->depart[k] < 0) return fail(h, SIM_E_INVALID, "depart_step must be >= 0" + id);
  }
  h->radj = radj;
  h->rstart.assign(nv, 0);
  h->rlen.assign(nv, 0);
  for (int k = 0; k < nv; ++k) { h->rstart[k] = h->route_off[k]; h->rlen[k] = h->route_off[k + 1] - h->route_off[k]; }
  h->P = *p;
  h->Y = p->yellow_steps;
  // batched environments (NEXT-3): per-vehicle Philox key / counter id, road groups
  if (p->vehicle_seed) h->vseed.assign(p->vehicle_seed, p->vehicle_seed + nv);
  if (p->vehicle_rng_id) {
    h->rngid.assign(p->vehicle_rng_id, p->vehicle_rng_id + nv);
    for (int k = 0; k < nv; ++k)
      if (h->rngid[k] < 0) return fail(h, SIM_E_INVALID, "vehicle_rng_id must be >= 0");
  }
  h->n_groups = 0;
  if (p->road_group) {
    if (p->n_groups < 1) return fail(h, SIM_E_INVALID, "n_groups must be >= 1 with road_group");
    h->n_groups = p->n_groups;
    h->road_group.assign(p->road_group, p->road_group + h->nr);
    for (int r = 0; r < h->nr; ++r)
      if (h->road_group[r] < 0 || h->road_group[r] >= p->n_groups)
        return fail(h, SIM_E_INVALID, "road_group out of [0, n_groups)");
    h->veh_group.assign(nv, 0);
    h->grp_nv.assign(h->n_groups, 0);
    for (int k = 0; k < nv; ++k) {
      h->veh_group[k] = h->road_group[h->road[h->start_lane[k]]];
      h->grp_nv[h->veh_group[k]] += 1;
    }
  }
  h->P.vehicle_seed = nullptr;                       // not retained (ABI: inputs are copied)
  h->P.vehicle_rng_id = nullptr;
  h->P.road_group = nullptr;
  h->profs.resize(p->n_profiles);
  float acap = 0;
  for (int i = 0; i < p->n_profiles; ++i) {
    const sim_profile &q = p->profiles[i];
    Prof &o = h->profs[i];
    o.a_max = q.a_max; o.a_comf = q.a_comf; o.T = q.T; o.s0 = q.s0; o.vmax = q.v_max; o.len = q.length;
    o.a_max_d = q.a_max; o.a_comf_d = q.a_comf; o.T_d = q.T; o.s0_d = q.s0; o.vmax_d = q.v_max; o.len_d = q.length;
    o.inv2sqrt_d = 1.0 / (2.0 * std::sqrt(o.a_max_d * o.a_comf_d));
    o.inv2sqrt_f = (float)o.inv2sqrt_d;
    o.pad = 0; o.pad_d = 0;
    acap = std::max(acap, q.a_max);
  }
  float vcap = 0;
  for (int l = 0; l < nl; ++l) vcap = std::max(vcap, h->vmax[l]);
  h->start_margin = (double)vcap + 0.5 * (double)acap;
  return SIM_OK;
}

sim_status build_tiles(sim_s *h) {
  // tile = road (leftmost lane first) + junction lanes whose predecessor is on it
  const int nr = h->nr, nl = h->nl;
  std::vector<std::vector<int>> jls(nr);
  for (int l = 0; l < nl; ++l)
    if (!is_road(h, l)) jls[h->road[h->pred[l]]].push_back(l);
  float lmin = 1e30f;
  for (auto &q : h->profs) lmin = std::min(lmin, q.len);
  h->nt = nr;
  h->tile_lane_off.assign(nr + 1, 0);
  h->tile_nroad.assign(nr, 0);
  h->lane_tile.assign(nl, -1);
  h->lane_local.assign(nl, 0);
  h->tile_lanes.clear();
  h->tile_base.assign(nr, 0); h->tile_cap.assign(nr, 0);
  h->tile_ibase.assign(nr, 0); h->tile_icap.assign(nr, 0);
  auto lane_cap = [&](int l) { return (int)std::floor(h->L[l] / lmin) + 2; };
  std::vector<int> feed(nr, 0);
  for (int l = 0; l < nl; ++l)
    for (int e = h->succ_off[l]; e < h->succ_off[l + 1]; ++e) {
      int j = h->succ[e];
      if (is_road(h, j) && h->lane_tile.size() && h->road[j] != (is_road(h, l) ? h->road[l] : h->road[h->pred[l]]))
        feed[h->road[j]] += lane_cap(l);
    }
  int64_t base = 0, ibase = 0;
  for (int r = 0; r < nr; ++r) {
    std::vector<int> lanes(h->road_lanes.begin() + h->road_off[r], h->road_lanes.begin() + h->road_off[r + 1]);
    h->tile_nroad[r] = (int)lanes.size();
    std::sort(jls[r].begin(), jls[r].end());
    lanes.insert(lanes.end(), jls[r].begin(), jls[r].end());
    if (h->tile_nroad[r] > kMaxRoadLanes)
      return fail(h, SIM_E_INVALID, "road " + std::to_string(r) + " has more than " +
                  std::to_string(kMaxRoadLanes) + " lanes");
    for (int q = 0; q < h->tile_nroad[r]; ++q) {
      const int l = lanes[q];
      std::vector<int> tr;
      for (int e = h->succ_off[l]; e < h->succ_off[l + 1]; ++e) tr.push_back(h->target_road[h->succ[e]]);
      std::sort(tr.begin(), tr.end());
      const int ntr = (int)(std::unique(tr.begin(), tr.end()) - tr.begin());
      if (h->succ_off[l + 1] - h->succ_off[l] > kMaxSucc || ntr > kMaxGroups)
        return fail(h, SIM_E_INVALID, "lane " + std::to_string(l) + " has more than " +
                    std::to_string(kMaxSucc) + " successors or " + std::to_string(kMaxGroups) +
                    " successor roads");
    }
    if ((int)lanes.size() > kMaxTileLanes)
      return fail(h, SIM_E_INVALID, "road " + std::to_string(r) + " has more than " + std::to_string(kMaxTileLanes) + " lanes incl. outgoing junction lanes");
    int cap = 0;
    for (size_t k = 0; k < lanes.size(); ++k) {
      h->lane_tile[lanes[k]] = r;
      h->lane_local[lanes[k]] = (uint8_t)k;
      h->tile_lanes.push_back(lanes[k]);
      cap += lane_cap(lanes[k]);
    }
    cap = (cap + cap / 4 + 16 + 3) & ~3;            // multiple of 4: 16-B aligned bulk copies
    int icap = cap + feed[r] + h->tile_nroad[r] + 16;
    if (cap > 32767 || icap > 32767)                // snapshot source indices are int16
      return fail(h, SIM_E_INVALID, "road " + std::to_string(r) + " is too long (tile capacity > 32767 vehicles)");
    h->tile_lane_off[r + 1] = (int)h->tile_lanes.size();
    // one record region per tile: stayers right-aligned in the
    // first cap slots, the inbox in the next icap
    h->tile_base[r] = (int)base; h->tile_cap[r] = cap;
    h->tile_ibase[r] = (int)(base + cap); h->tile_icap[r] = icap;
    base += cap + icap;
    if (base > 2000000000LL) return fail(h, SIM_E_INVALID, "network too large for 32-bit slot indices");
  }
  h->n_slots = base;
  return SIM_OK;
}

// initial signal state: FIXED_TIME advanced `offset` steps
void init_junctions(sim_s *h, HostState &S) {
  S.jpol.assign(h->nj, 0); S.jphase.assign(h->nj, 0); S.jel.assign(h->nj, 0);
  S.jy.assign(h->nj, 0); S.jpend.assign(h->nj, 0); S.jrem.assign(h->nj, -1);
  for (int j = 0; j < h->nj; ++j) {
    int K = h->ph_off[j + 1] - h->ph_off[j];
    int pol = K == 0 ? POL_NONE : h->pol0[j];
    int ph = 0, el = 0, y = 0, q = 0;
    if (pol == POL_FIXED)
      for (int s = 0; s < h->offset0[j]; ++s) {
        if (y > 0) { y -= 1; if (y == 0) { ph = q; el = 0; } }
        else {
          el += 1;
          if (el >= h->green_steps[h->ph_off[j] + ph]) {
            int nx = (ph + 1) % K;
            if (h->Y > 0) { y = h->Y; q = nx; } else { ph = nx; q = nx; el = 0; }
          }
        }
      }
    S.jpol[j] = (uint8_t)pol; S.jphase[j] = ph; S.jel[j] = el; S.jy[j] = y; S.jpend[j] = q;
  }
}


int route_at(const sim_s *h, int vid, int idx) {
  int a = h->rstart[vid], n = h->rlen[vid];
  return (idx >= 0 && idx < n) ? h->route[a + idx] : -1;
}

// ---- partitioning ---------------------------------------------
// Default partitioner: breadth-first order of the roads over the undirected
// road adjacency (deterministic, from road 0, ties by id), cut into `world`
// contiguous chunks of equal slot capacity.  Callers with coordinates can pass
// their own road_owner (bench.py uses recursive coordinate bisection).
std::vector<int> default_partition(const sim_s *h, int world,
                                   const std::vector<int64_t> *weight = nullptr) {
  std::vector<std::vector<int>> adj(h->nr);
  for (int l = 0; l < h->nl; ++l) {
    if (!is_road(h, l)) continue;
    for (int e = h->succ_off[l]; e < h->succ_off[l + 1]; ++e) {
      int r1 = h->road[l], r2 = h->target_road[h->succ[e]];
      if (r1 != r2) { adj[r1].push_back(r2); adj[r2].push_back(r1); }
    }
  }
  for (auto &a : adj) { std::sort(a.begin(), a.end()); a.erase(std::unique(a.begin(), a.end()), a.end()); }
  std::vector<int> order;
  std::vector<char> seen(h->nr, 0);
  for (int s = 0; s < h->nr; ++s) {
    if (seen[s]) continue;
    std::deque<int> q{s};
    seen[s] = 1;
    while (!q.empty()) {
      int r = q.front(); q.pop_front();
      order.push_back(r);
      for (int x : adj[r]) if (!seen[x]) { seen[x] = 1; q.push_back(x); }
    }
  }
  // weight of a road tile: its slot capacity, or (repartition) the given load
  auto wt = [&](int r) { return weight ? (*weight)[r] : (int64_t)h->tile_cap[r]; };
  int64_t tot = 0;
  for (int r = 0; r < h->nr; ++r) tot += wt(r);
  std::vector<int> owner(h->nr, 0);
  int64_t acc = 0;
  for (int r : order) {
    owner[r] = (int)std::min<int64_t>(world - 1, (acc * world) / std::max<int64_t>(tot, 1));
    acc += wt(r);
  }
  return owner;
}

// Exchange plan: migrant capacities and halo lane lists for every ordered pair.
struct Plan {
  std::vector<std::vector<int>> mig_cap;             // [from][to]
  std::vector<std::vector<std::vector<int>>> halo;   // [reader][owner] sorted lanes
};

Plan make_plan(const sim_s *h) {
  const int W = h->world;
  Plan P;
  P.mig_cap.assign(W, std::vector<int>(W, 0));
  P.halo.assign(W, std::vector<std::vector<int>>(W));
  float lmin = 1e30f, acap = 0, vcap = 0;
  for (auto &q : h->profs) { lmin = std::min(lmin, q.len); acap = std::max(acap, q.a_max); }
  for (int l = 0; l < h->nl; ++l) vcap = std::max(vcap, h->vmax[l]);
  const int reach = (int)std::ceil((vcap + acap) / lmin) + 2;   // vehicles within one step of a lane end
  auto owner_of = [&](int l) { return h->tile_owner[h->lane_tile[l]]; };
  for (int l = 0; l < h->nl; ++l) {
    const int a = owner_of(l);
    for (int e = h->succ_off[l]; e < h->succ_off[l + 1]; ++e) {
      const int y = h->succ[e], b = owner_of(y);
      if (a == b) continue;
      // a vehicle can leave through y only from l (or from l's predecessor road
      // lane in the same step when l is a short junction lane)
      int c = (int)std::floor(h->L[l] / lmin) + 2 + reach;
      P.mig_cap[a][b] += c;
    }
  }
  for (int a = 0; a < W; ++a)
    for (int b = 0; b < W; ++b)
      if (P.mig_cap[a][b]) P.mig_cap[a][b] = 2 * P.mig_cap[a][b] + 64;
  // halo: lanes within `lookahead` successor hops of a lane owned by the reader
  const int K = std::max(h->P.lookahead_lanes, 1);
  std::vector<std::set<int>> need(W);
  for (int l = 0; l < h->nl; ++l) {
    const int a = owner_of(l);
    std::vector<int> front{l};
    for (int hop = 0; hop < K; ++hop) {
      std::vector<int> nxt;
      for (int x : front)
        for (int e = h->succ_off[x]; e < h->succ_off[x + 1]; ++e) {
          int y = h->succ[e];
          nxt.push_back(y);
          if (owner_of(y) != a) need[a].insert(y);
        }
      front.swap(nxt);
    }
  }
  for (int a = 0; a < W; ++a)
    for (int y : need[a]) P.halo[a][owner_of(y)].push_back(y);
  return P;
}

sim_status push_staging(sim_s *h, const void *src, size_t bytes, void *dst) {
  if (bytes == 0) return SIM_OK;
  if (h->pinned_cap < bytes) {
    if (h->pinned) { CK(h, cudaEventSynchronize(h->stage_ev)); cudaFreeHost(h->pinned); }
    h->pinned = nullptr;
    CK(h, cudaHostAlloc(&h->pinned, bytes, cudaHostAllocDefault));
    h->pinned_cap = bytes;
  } else {
    CK(h, cudaEventSynchronize(h->stage_ev));
  }
  std::memcpy(h->pinned, src, bytes);
  CK(h, cudaMemcpyAsync(dst, h->pinned, bytes, cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaEventRecord(h->stage_ev, h->stream));
  return SIM_OK;
}

// Upload a full state (canonical: stayer slabs sorted per lane, empty inboxes)
// into every partition; each keeps the vehicles of its own tiles, all other
// state (summaries, cold arrays, signals, queues) is replicated.
sim_status read_counters(sim_s *h, std::vector<long long> &out);
sim_status read_group_counters(sim_s *h, std::vector<long long> &c);

sim_status upload_state(sim_s *h, const HostState &S) {
  const int nv = h->nv, nt = h->nt, t = S.t;
  const int par = t & 1;
  h->t = t;
  h->dir = S.dir;
  compute_usable(h);
  std::vector<std::vector<int>> per_tile(nt), in_tile(nt);
  for (int k = 0; k < nv; ++k)
    if (S.status[k] == ST_DRIVING) {
      int l = S.lane[k];
      if (l < 0 || l >= h->nl) return fail(h, SIM_E_RANGE, "lane out of range for driving vehicle " + std::to_string(k));
      if (!S.to_inbox.empty() && S.to_inbox[k]) in_tile[h->lane_tile[l]].push_back(k);
      else per_tile[h->lane_tile[l]].push_back(k);
    }
  std::vector<InboxRec> rec(h->n_slots);
  std::memset(rec.data(), 0, rec.size() * sizeof(InboxRec));
  std::vector<int> cnt(nt, 0), icnt(nt, 0);
  std::vector<unsigned long long> summ(h->nl, kEmptyKey);
  std::vector<float> pubv(nv, 0.f);
  for (int T = 0; T < nt; ++T) {
    auto &ks = per_tile[T];
    std::sort(ks.begin(), ks.end(), [&](int a, int b) {
      int la = h->lane_local[S.lane[a]], lb = h->lane_local[S.lane[b]];
      if (la != lb) return la < lb;
      if (S.s[a] != S.s[b]) return S.s[a] < S.s[b];
      return a < b;
    });
    if ((int)ks.size() > h->tile_cap[T])
      return fail(h, SIM_E_CAPACITY, "state exceeds the slot capacity of road tile " + std::to_string(T));
    const int p0 = h->tile_base[T] + h->tile_cap[T] - (int)ks.size();   // right-aligned stayers
    for (size_t i = 0; i < ks.size(); ++i) {
      int k = ks[i];
      InboxRec &r = rec[(size_t)p0 + i];
      r.s = S.s[k] == 0.0f ? 0.0f : S.s[k];
      r.v = S.v[k];
      r.vid = k;
      r.nxt = route_at(h, k, S.cursor[k] + 1);
      r.nxt2 = route_at(h, k, S.cursor[k] + 2);
      r.meta = pack_meta(h->lane_local[S.lane[k]], h->vprof[k], S.cursor[k]);
      r.wait = S.wait[k];
      r.end_s = h->end_s[k];
      unsigned long long key = ((unsigned long long)*(const uint32_t *)&r.s << 32) | (unsigned)k;
      int l = S.lane[k];
      if (key < summ[l]) summ[l] = key;
      pubv[k] = S.v[k];
    }
    cnt[T] = (int)ks.size();
    // test hook: the rest of the tile's vehicles as unsorted inbox records
    // (reverse vid order), as if they had entered or changed lane in step t-1
    auto &ib = in_tile[T];
    std::sort(ib.rbegin(), ib.rend());
    if ((int)ib.size() > h->tile_icap[T])
      return fail(h, SIM_E_CAPACITY, "state exceeds the inbox capacity of road tile " + std::to_string(T));
    for (size_t i = 0; i < ib.size(); ++i) {
      const int k = ib[i];
      InboxRec &r = rec[(size_t)h->tile_ibase[T] + i];
      r.s = S.s[k] == 0.0f ? 0.0f : S.s[k];
      r.v = S.v[k];
      r.vid = k;
      r.nxt = route_at(h, k, S.cursor[k] + 1);
      r.nxt2 = route_at(h, k, S.cursor[k] + 2);
      r.meta = pack_meta(h->lane_local[S.lane[k]], h->vprof[k], S.cursor[k]);
      r.wait = S.wait[k];
      r.end_s = h->end_s[k];
      unsigned long long key = ((unsigned long long)*(const uint32_t *)&r.s << 32) | (unsigned)k;
      int l = S.lane[k];
      if (key < summ[l]) summ[l] = key;
      pubv[k] = S.v[k];
    }
    icnt[T] = (int)ib.size();
  }
  std::vector<int> wfin(nv, 0);
  h->fin0 = 0;
  h->ins0 = 0;
  for (int k = 0; k < nv; ++k) {
    wfin[k] = S.status[k] == ST_FINISHED ? S.wait[k] : 0;
    h->fin0 += S.status[k] == ST_FINISHED;
    if (S.status[k] == ST_DRIVING) h->ins0 += S.insert_time[k];
  }
  // pending queues per start lane sorted by (depart, vid) (ledger L25)
  std::vector<std::vector<int>> pq(h->nl);
  for (int k = 0; k < nv; ++k)
    if (S.status[k] == ST_PENDING) pq[h->start_lane[k]].push_back(k);
  std::vector<int> poff(h->nl + 1, 0), pvid;
  for (int l = 0; l < h->nl; ++l) {
    std::sort(pq[l].begin(), pq[l].end(), [&](int a, int b) {
      return h->depart[a] != h->depart[b] ? h->depart[a] < h->depart[b] : a < b;
    });
    poff[l + 1] = poff[l] + (int)pq[l].size();
    pvid.insert(pvid.end(), pq[l].begin(), pq[l].end());
  }
  std::vector<int> head(poff.begin(), poff.end() - 1);
  std::vector<int> req(h->nj, -1);
  // MAX_PRESSURE lane counts of state(t) (L39)
  h->any_maxp = false;
  for (int j = 0; j < h->nj; ++j) h->any_maxp |= S.jpol[j] == POL_MAXP;
  {
    std::vector<int32_t> lc(h->nl, 0);
    for (int k = 0; k < nv; ++k)
      if (S.status[k] == ST_DRIVING) lc[S.lane[k]] += 1;
    CK(h, cudaMemcpyAsync(h->lcnt[t % 3], lc.data(), h->nl * 4, cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaMemsetAsync(h->lcnt[(t + 1) % 3], 0, h->nl * 4, h->stream));
    CK(h, cudaMemsetAsync(h->lcnt[(t + 2) % 3], 0, h->nl * 4, h->stream));
  }
  for (Part &P : h->parts) {
    cudaStream_t st = h->stream;
    std::vector<int> pc(nt, 0), pic(nt, 0);
    for (int T : P.tiles) { pc[T] = cnt[T]; pic[T] = icnt[T]; }
    CK(h, cudaMemcpyAsync(P.usable_d, h->usable.data(), h->nl, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.outroads_d, h->outroads.data(), h->outroads.size() * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.desc_d, h->desc.data(), h->desc.size() * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.inbox[par], rec.data(), rec.size() * sizeof(InboxRec), cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.cnt[par], pc.data(), nt * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemsetAsync(P.icnt[par ^ 1], 0, nt * 4, st));
    CK(h, cudaMemcpyAsync(P.icnt[par], pic.data(), nt * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.summ[t % 3], summ.data(), h->nl * 8, cudaMemcpyHostToDevice, st));
    launch_fill_u64(P.summ[(t + 1) % 3], kEmptyKey, h->nl, st);
    launch_fill_u64(P.summ[(t + 2) % 3], kEmptyKey, h->nl, st);
    CK(h, cudaMemcpyAsync(P.pubv[par], pubv.data(), nv * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.A.status, S.status.data(), nv, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.A.insert_time, S.insert_time.data(), nv * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.A.arrive_time, S.arrive_time.data(), nv * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.A.wait_fin, wfin.data(), nv * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.pend_off_d, poff.data(), poff.size() * 4, cudaMemcpyHostToDevice, st));
    if (!pvid.empty())
      CK(h, cudaMemcpyAsync(P.pend_vid_d, pvid.data(), pvid.size() * 4, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(P.pend_head_d, head.data(), head.size() * 4, cudaMemcpyHostToDevice, st));
    if (h->nj) {
      CK(h, cudaMemcpyAsync(P.SG.policy, S.jpol.data(), h->nj, cudaMemcpyHostToDevice, st));
      CK(h, cudaMemcpyAsync(P.SG.phase, S.jphase.data(), h->nj * 4, cudaMemcpyHostToDevice, st));
      CK(h, cudaMemcpyAsync(P.SG.elapsed, S.jel.data(), h->nj * 4, cudaMemcpyHostToDevice, st));
      CK(h, cudaMemcpyAsync(P.SG.yellow_left, S.jy.data(), h->nj * 4, cudaMemcpyHostToDevice, st));
      CK(h, cudaMemcpyAsync(P.SG.pending, S.jpend.data(), h->nj * 4, cudaMemcpyHostToDevice, st));
      CK(h, cudaMemcpyAsync(P.SG.remaining, S.jrem.data(), h->nj * 4, cudaMemcpyHostToDevice, st));
      CK(h, cudaMemcpyAsync(P.SG.dur_request, req.data(), h->nj * 4, cudaMemcpyHostToDevice, st));
      CK(h, cudaMemcpyAsync(P.SG.request, req.data(), h->nj * 4, cudaMemcpyHostToDevice, st));
      CK(h, cudaMemcpyAsync(P.SG.pol_request, req.data(), h->nj * 4, cudaMemcpyHostToDevice, st));
    }
    if (P.out_cnt) CK(h, cudaMemsetAsync(P.out_cnt, 0, h->world * 4, st));
  }
  CK(h, cudaStreamSynchronize(h->stream));   // host vectors die at return
  // counters keep accumulating across loads: remember the finished baseline,
  // reduced exactly as sim_read_metrics / sim_read_group_metrics reduce them
  // (all tiles of every partition, summed across processes), so that
  // n_finished stays the loaded count plus the arrivals since on every rank
  h->acc_fin0 = 0;
  h->acc_ins0 = 0;
  h->grp_fin0.assign(h->n_groups, 0);
  h->grp_acc_fin0.assign(h->n_groups, 0);
  for (int k = 0; k < nv && h->n_groups; ++k) h->grp_fin0[h->veh_group[k]] += S.status[k] == ST_FINISHED;
  if (!(h->ipc && !h->connected)) {                // (before sim_ipc_connect every counter is 0)
    std::vector<long long> c;
    sim_status st = read_counters(h, c);
    if (st) return st;
    h->acc_fin0 = c[ACC_FINISHED];
    h->acc_ins0 = c[ACC_SUM_INSERT];
    if (h->n_groups) {
      st = read_group_counters(h, c);
      if (st) return st;
      for (int g = 0; g < h->n_groups; ++g) h->grp_acc_fin0[g] = c[(size_t)g * (kNAcc + 1) + ACC_FINISHED];
    }
  }
  return SIM_OK;
}

sim_status alloc_part(sim_s *h, Part &P, const Plan *plan) {
  sim_status st;
#define AL(p, n) if ((st = dalloc(h, &(p), (n)))) return st
#define UP(p, v) if ((st = upload(h, &(p), (v)))) return st
  StepArgs &A = P.A;
  const int nl = h->nl, nv = h->nv, nt = h->nt;
  float *f; int32_t *i32;
  UP(f, h->L); A.lane_len = f;
  UP(f, h->vmax); A.lane_vmax = f; P.lane_vmax_d = f;
  UP(i32, h->road); A.lane_road = i32;
  UP(i32, h->left); A.lane_left = i32;
  UP(i32, h->right); A.lane_right = i32;
  UP(i32, h->succ_off); A.succ_off = i32;
  UP(i32, h->succ); A.succ = i32;
  UP(i32, h->target_road); A.target_road = i32;
  UP(i32, h->exit_lane); A.exit_lane = i32;
  AL(P.usable_d, nl); A.usable = P.usable_d;
  AL(P.outroads_d, 4 * (size_t)nl); A.outroads = reinterpret_cast<const int4 *>(P.outroads_d);
  AL(P.desc_d, h->desc.size()); A.desc = P.desc_d;
  UP(i32, h->desc_off); A.desc_off = i32;
  uint8_t *sig; AL(sig, nl);
  CK(h, dmemset(h, sig, 0, nl));
  A.lane_sig = sig;
  UP(i32, h->lane_tile); A.lane_tile = i32;
  uint8_t *u8; UP(u8, h->lane_local); A.lane_local = u8;
  UP(i32, h->tile_lane_off); A.tile_lane_off = i32;
  UP(i32, h->tile_lanes); A.tile_lanes = i32;
  UP(i32, h->tile_nroad); A.tile_nroad = i32;
  UP(i32, h->tile_base); A.tile_base = i32;
  UP(i32, h->tile_cap); A.tile_cap = i32;
  UP(i32, h->tile_ibase); A.tile_ibase = i32;
  UP(i32, h->tile_icap); A.tile_icap = i32;
  UP(i32, h->tile_owner); A.tile_owner = i32;
  {
    // largest tiles first: the persistent step kernel takes tiles in this order
    std::vector<int> order(P.tiles);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return h->tile_cap[a] > h->tile_cap[b]; });
    UP(i32, order); A.tiles = i32;
  }
  AL(A.work, 2);
  CK(h, dmemset(h, A.work, 0, 8));
  AL(A.bk_cnt, kNBucket);
  CK(h, dmemset(h, A.bk_cnt, 0, kNBucket * 4));
  AL(A.bk_list, (size_t)kNBucket * nt);
  A.n_own = (int)P.tiles.size();
  A.rank = P.rank;
  for (int b = 0; b < 2; ++b) {
    AL(P.inbox[b], h->n_slots);                   // vehicle records: stayers + inboxes
    AL(P.cnt[b], nt); AL(P.icnt[b], nt);
    AL(P.pubv[b], nv);
    CK(h, dmemset(h, P.cnt[b], 0, nt * 4));
    CK(h, dmemset(h, P.icnt[b], 0, nt * 4));
    CK(h, dmemset(h, P.pubv[b], 0, nv * 4));
  }
  const int64_t sc = h->n_slots;
  AL(A.scratch, 8 * sc);
  AL(A.bsort_scratch, sc);
  AL(A.pscratch, 10 * (sc + 4 * (int64_t)nt));
  {
    // static per-tile record read by k_step's producer warp and k_prep
    std::vector<int4> ti(3 * (size_t)nt);
    for (int T = 0; T < nt; ++T) {
      const int nlT = h->tile_lane_off[T + 1] - h->tile_lane_off[T], nr = h->tile_nroad[T];
      ti[3 * T + 0] = make_int4(h->tile_base[T], h->tile_ibase[T], h->tile_cap[T], h->tile_icap[T]);
      ti[3 * T + 1] = make_int4(h->desc_off[T], h->desc_off[T + 1] - h->desc_off[T], nlT, nr);
      ti[3 * T + 2] = make_int4(h->desc_words[T], 0, 0, 0);
    }
    int4 *i4; UP(i4, ti); A.tinfo = i4;
  }
  for (int b = 0; b < 3; ++b) AL(P.summ[b], nl);
  UP(P.route_start_d, h->rstart); A.route_start = P.route_start_d;
  UP(P.route_len_d, h->rlen); A.route_len = P.route_len_d;
  if (!h->route_cap) h->route_cap = (int64_t)h->route.size() + (int64_t)h->route.size() / 4 + 4096;
  AL(P.route_d, h->route_cap); A.route = P.route_d;
  CK(h, cudaMemcpy(P.route_d, h->route.data(), h->route.size() * 4, cudaMemcpyHostToDevice));
  UP(f, h->end_s); A.end_s = f; P.end_s_d = f;
  AL(P.patch_d, nv);
  CK(h, dmemset(h, P.patch_d, 0xff, (size_t)nv * 4));
  UP(u8, h->vprof); A.veh_prof = u8;
  AL(A.insert_time, nv); AL(A.arrive_time, nv); AL(A.wait_fin, nv); AL(A.status, nv);
  UP(i32, h->depart); A.depart = i32;
  UP(f, h->start_s); A.start_s = f;
  AL(P.pend_off_d, nl + 1); AL(P.pend_vid_d, nv); AL(P.pend_head_d, nl);
  A.pend_off = P.pend_off_d; A.pend_vid = P.pend_vid_d; A.pend_head = P.pend_head_d;
  Prof *pr; UP(pr, h->profs); A.prof = pr;
  A.veh_seed = nullptr;
  A.rng_id = nullptr;
  if (!h->vseed.empty()) { uint64_t *u64; UP(u64, h->vseed); A.veh_seed = u64; }
  if (!h->rngid.empty()) { UP(i32, h->rngid); A.rng_id = i32; }
  if (h->n_groups) {
    UP(P.tile_group_d, h->road_group);               // tile = road
    AL(P.grp_d, (size_t)h->n_groups * (kNAcc + 1));
  }
  AL(A.tacc, (size_t)nt * kNAcc);
  CK(h, dmemset(h, A.tacc, 0, (size_t)nt * kNAcc * 8));
  AL(P.red_d, kNAcc + 3);
  AL(P.lanestat_d, 2 * (size_t)nl + h->nr);           // lane counts, waiting, road speeds
  if (h->world > 1 && !h->loopback) AL(P.xch_d, 3 * (size_t)nv + 8);   // one process per rank
  if (h->P.record_decisions) {
    AL(A.r_leader, nv); AL(A.r_of, nv); AL(A.r_side, 4 * (size_t)nv);
    AL(A.r_hops, nv); AL(A.r_phantom, nv); AL(A.r_lc, nv); AL(A.r_hand, nv);
    AL(A.r_fin, nv); AL(A.r_ins, nv); AL(A.r_acc, nv); AL(A.r_guard, nv); AL(A.r_mark, nv);
  }
  // exchange buffers
  const int W = h->world;
  if (W > 1 && plan) {
    P.out_off.assign(W + 1, 0); P.out_cap.assign(W, 0);
    P.in_off.assign(W + 1, 0); P.in_cap.assign(W, 0);
    for (int q = 0; q < W; ++q) {
      P.out_cap[q] = plan->mig_cap[P.rank][q];
      P.in_cap[q] = plan->mig_cap[q][P.rank];
      P.out_off[q + 1] = P.out_off[q] + (P.out_cap[q] ? P.out_cap[q] + 1 : 0);
      P.in_off[q + 1] = P.in_off[q] + (P.in_cap[q] ? P.in_cap[q] + 1 : 0);
    }
    P.out_n = P.out_off[W]; P.in_n = P.in_off[W];
    AL(P.out_buf, P.out_n); AL(P.in_buf, P.in_n); AL(P.out_cnt, W);
    CK(h, dmemset(h, P.out_cnt, 0, W * 4));
    CK(h, dmemset(h, P.in_buf, 0, std::max<int64_t>(P.in_n, 1) * sizeof(MigRec)));
    std::vector<int> off(P.out_off.begin(), P.out_off.end() - 1);
    UP(i32, off); A.out_off = i32;
    UP(i32, P.out_cap); A.out_cap = i32;
    std::vector<int> ioff(P.in_off.begin(), P.in_off.end() - 1);
    UP(P.in_off_d, ioff);
    UP(P.in_cap_d, P.in_cap);
    A.out_buf = P.out_buf; A.out_cnt = P.out_cnt;
    std::vector<int> hs, hr;
    P.hs_off.assign(W + 1, 0); P.hr_off.assign(W + 1, 0);
    for (int q = 0; q < W; ++q) {
      const auto &snd = plan->halo[q][P.rank];      // lanes peer q reads from us
      const auto &rcv = plan->halo[P.rank][q];      // lanes we read from q
      hs.insert(hs.end(), snd.begin(), snd.end());
      hr.insert(hr.end(), rcv.begin(), rcv.end());
      P.hs_off[q + 1] = (int)hs.size();
      P.hr_off[q + 1] = (int)hr.size();
    }
    P.hs_n = (int64_t)hs.size(); P.hr_n = (int64_t)hr.size();
    UP(P.hs_lanes, hs); UP(P.hr_lanes, hr);
    AL(P.hs_buf, P.hs_n); AL(P.hr_buf, P.hr_n);
  }
  if (h->direct) {
    AL(P.bar_d, 1);
    CK(h, dmemset(h, P.bar_d, 0, 4));
  }
  // signals (replicated: every partition runs every junction's controller)
  SignalArgs &G = P.SG;
  G.n_junctions = h->nj; G.yellow = h->Y;
  AL(G.policy, h->nj); AL(G.phase, h->nj); AL(G.elapsed, h->nj); AL(G.yellow_left, h->nj);
  AL(G.pending, h->nj); AL(G.request, h->nj); AL(G.pol_request, h->nj);
  AL(G.remaining, h->nj); AL(G.dur_request, h->nj);
  UP(i32, h->jl_off); G.jl_off = i32;
  UP(i32, h->jl); G.jl = i32;
  UP(i32, h->ph_off); G.ph_off = i32;
  int64_t *g64; UP(g64, h->green_off); G.green_off = g64;
  UP(u8, h->green); G.green = u8;
  UP(i32, h->green_steps); G.green_steps = i32;
  G.lane_sig = sig;
  UP(i32, h->jl_pred); G.jl_pred = i32;
  UP(i32, h->jl_succ); G.jl_succ = i32;
  G.mp_period = h->P.max_pressure_period > 0 ? h->P.max_pressure_period : 30;
  if (!h->lcnt[0])                                  // shared by loopback partitions
    for (int b = 0; b < 3; ++b) { AL(h->lcnt[b], nl); CK(h, dmemset(h, h->lcnt[b], 0, nl * 4)); }
  // constants
  A.n_tiles = nt; A.n_lanes = nl; A.n_veh = nv;
  A.seed = h->P.seed;
  A.polite = h->P.politeness; A.b_hard = h->P.b_hard; A.b_safe = h->P.b_safe; A.v_wait = h->P.v_wait;
  A.start_margin = h->start_margin;
  A.lookahead = h->P.lookahead_lanes;
  A.exact_mode = h->P.exact_mode;
  A.record = h->P.record_decisions;
  A.n_prof = (int)h->profs.size();
  A.peers = nullptr;
  G.peers = nullptr;
  G.lane_tile = A.lane_tile;
  G.tile_owner = A.tile_owner;
  PeerView &V = P.view;
  for (int b = 0; b < 2; ++b) { V.inbox[b] = P.inbox[b]; V.icnt[b] = P.icnt[b]; V.pubv[b] = P.pubv[b]; }
  for (int b = 0; b < 3; ++b) { V.summ[b] = P.summ[b]; V.lcnt[b] = h->lcnt[b]; }
  V.insert_time = A.insert_time;
  V.status = A.status;
  V.bar = P.bar_d;
  for (int b = 0; b < 2; ++b) V.cnt[b] = P.cnt[b];
  V.pend_head = P.pend_head_d;
  V.arrive_time = A.arrive_time;
  V.wait_fin = A.wait_fin;
  V.xbuf[0] = P.red_d;
  V.xbuf[1] = P.lanestat_d;
  V.xbuf[2] = P.grp_d;
  V.xbuf[3] = P.xch_d;
  return SIM_OK;
#undef AL
#undef UP
}

StepArgs step_args(const Part &P, int t) {
  StepArgs a = P.A;
  const int par = t & 1;
  a.t = t;
  a.cnt_in = P.cnt[par];
  a.cnt_out = P.cnt[par ^ 1];
  a.icnt_in = P.icnt[par];
  a.icnt_out = P.icnt[par ^ 1];
  a.vin = P.inbox[par];
  a.vout = P.inbox[par ^ 1];
  a.summ_cur = P.summ[t % 3];
  a.summ_next = P.summ[(t + 1) % 3];
  a.summ_clear = P.summ[(t + 2) % 3];
  a.pubv_cur = P.pubv[par];
  a.pubv_next = P.pubv[par ^ 1];
  a.lane_cnt_next = nullptr;
  return a;
}

sim_status check(sim_s *h) {
  if (!h || !is_live(h)) return fail(nullptr, SIM_E_STATE, "null or destroyed handle");
  if (h->sticky) return fail(h, SIM_E_STATE, "handle is in a sticky error state: " + h->err);
  // every call works on the handle's device (allocations, launches, IPC
  // mappings), whatever device the calling thread had current
  if (cudaSetDevice(h->device) != cudaSuccess) return fail(h, SIM_E_CUDA, "cudaSetDevice failed");
  return SIM_OK;
}

sim_status device_check(sim_s *h) {
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    h->sticky = SIM_E_CUDA;
    return fail(h, SIM_E_CUDA, std::string("CUDA (deferred): ") + cudaGetErrorString(e));
  }
  if (h->bar_err_d) {
    int32_t be = 0;
    if (cudaMemcpy(&be, h->bar_err_d, 4, cudaMemcpyDeviceToHost) == cudaSuccess && be) {
      h->sticky = SIM_E_STATE;
      return fail(h, SIM_E_STATE, "direct transport: a peer barrier timed out (a peer stopped stepping)");
    }
  }
  return SIM_OK;
}

// Direct transport (NEXT-2): the table of every partition's buffers.  In one
// process it is complete at create; across processes this rank's own entry is
// filled now and the peers' by sim_ipc_connect.
sim_status upload_peers(sim_s *h, const std::vector<PeerView> &views) {
  for (Part &P : h->parts) {
    if (!P.peers_d) {
      sim_status st = dalloc(h, &P.peers_d, (size_t)h->world);
      if (st) return st;
    }
    CK(h, cudaMemcpy(P.peers_d, views.data(), views.size() * sizeof(PeerView), cudaMemcpyHostToDevice));
    P.A.peers = P.peers_d;
    P.SG.peers = P.peers_d;
  }
  return SIM_OK;
}

sim_status setup_direct(sim_s *h) {
  if (!h->ipc) {
    std::vector<PeerView> v;
    for (Part &P : h->parts) v.push_back(P.view);
    return upload_peers(h, v);
  }
  if (h->P.barrier_timeout_ms > 0) h->bar_timeout_ns = (unsigned long long)h->P.barrier_timeout_ms * 1000000ull;
  sim_status st = dalloc(h, &h->bar_err_d, 1);
  if (st) return st;
  CK(h, dmemset(h, h->bar_err_d, 0, 4));
  const size_t tmp = std::max<size_t>({(size_t)(kNAcc + 3) * 8, (2 * (size_t)h->nl + h->nr) * 4,
                                       (size_t)h->n_groups * (kNAcc + 1) * 8});
  char *t = nullptr;
  st = dalloc(h, &t, tmp);
  h->ipc_tmp = t;
  return st;
}

// The exported buffers of a PeerView, in a fixed order (sim_ipc_export).
constexpr int kIpcBufs = (int)(sizeof(PeerView) / sizeof(void *));
static_assert(sizeof(PeerView) == kIpcBufs * sizeof(void *), "PeerView holds pointers only");
void **view_slot(PeerView &V, int k) { return reinterpret_cast<void **>(&V) + k; }

// Direct transport across processes (NEXT-2): a device barrier over all
// partitions, stream-ordered.
sim_status barrier(sim_s *h) {
  if (!h->ipc) return SIM_OK;
  if (!h->connected) return fail(h, SIM_E_STATE, "direct transport: sim_ipc_connect has not been called");
  h->bar_epoch += 1;
  launch_barrier(h->parts[0].peers_d, h->world, h->rank, h->bar_epoch * (unsigned)h->world,
                 h->bar_err_d, h->bar_timeout_ns, h->stream);
  h->n_launch++;
  return SIM_OK;
}

// Sum over ranks of a read-side buffer (xbuf[kind] + off, n elements of
// dtype 0 int64 / 1 int32 / 2 float32): ncclAllReduce, or with the direct
// transport a peer-memory sum between two barriers.
sim_status allreduce_sum(sim_s *h, int kind, int dtype, int64_t off, int64_t n) {
  Part &P = h->parts[0];
  char *buf = reinterpret_cast<char *>(P.view.xbuf[kind]) + off * (dtype == 0 ? 8 : 4);
  if (h->comm) {
    const int nd = dtype == 0 ? kNcclInt64 : (dtype == 1 ? 2 /*ncclInt32*/ : 7 /*ncclFloat32*/);
    NK(h, g_nccl.AllReduce(buf, buf, n, nd, kNcclSum, h->comm, h->stream));
  } else if (h->ipc) {
    sim_status st = barrier(h);                     // every rank's contribution is written
    if (st) return st;
    launch_peer_sum(P.peers_d, h->world, kind, dtype, off, n, h->ipc_tmp, h->stream);
    h->n_launch++;
    st = barrier(h);                                // every rank has read ours
    if (st) return st;
    CK(h, cudaMemcpyAsync(buf, h->ipc_tmp, n * (dtype == 0 ? 8 : 4), cudaMemcpyDeviceToDevice, h->stream));
  }
  return SIM_OK;
}

// Global int64 counters: per-partition reduction, summed over loopback
// partitions / ncclAllReduce'd over ranks.
sim_status read_counters(sim_s *h, std::vector<long long> &out) {
  out.assign(kNAcc + 3, 0);
  for (Part &P : h->parts) {
    StepArgs a = step_args(P, h->t);
    launch_reduce_acc(P.A.tacc, h->nt, a.cnt_in, a.icnt_in, P.A.status, 0, P.red_d, h->stream);
    h->n_launch += 1;
  }
  if (h->comm || h->ipc) {
    sim_status st = allreduce_sum(h, 0, 0, 0, kNAcc + 3);
    if (st) return st;
  }
  std::vector<long long> tmp(kNAcc + 3);
  for (Part &P : h->parts) {
    CK(h, cudaMemcpyAsync(tmp.data(), P.red_d, (kNAcc + 3) * 8, cudaMemcpyDeviceToHost, h->stream));
    sim_status st = device_check(h);
    if (st) return st;
    for (int c = 0; c < kNAcc + 3; ++c) out[c] += tmp[c];
  }
  if (out[ACC_OVERFLOW] > 0) {
    h->sticky = SIM_E_CAPACITY;
    return fail(h, SIM_E_CAPACITY, "a road-tile inbox or a migration buffer overflowed its capacity");
  }
  return SIM_OK;
}

// Per-group counters [n_groups][kNAcc + 1], summed over the partitions the
// same way as read_counters (collective across processes).
sim_status read_group_counters(sim_s *h, std::vector<long long> &c) {
  const size_t w = (size_t)h->n_groups * (kNAcc + 1);
  c.assign(w, 0);
  std::vector<long long> tmp(w);
  for (Part &P : h->parts) {
    StepArgs a = step_args(P, h->t);
    launch_reduce_groups(P.A.tacc, h->nt, P.A.tiles, P.A.n_own, P.tile_group_d, a.cnt_in, a.icnt_in,
                         h->n_groups, P.grp_d, h->stream);
    h->n_launch += 1;
  }
  if (h->comm || h->ipc) {
    sim_status st = allreduce_sum(h, 2, 0, 0, (int64_t)w);
    if (st) return st;
  }
  for (size_t q = 0; q < h->parts.size(); ++q) {
    CK(h, cudaMemcpyAsync(tmp.data(), h->parts[q].grp_d, w * 8, cudaMemcpyDeviceToHost, h->stream));
    sim_status st = device_check(h);
    if (st) return st;
    for (size_t i = 0; i < w; ++i) c[i] += tmp[i];
    if (h->comm || h->ipc) break;                     // allreduced: one copy holds the total
  }
  return SIM_OK;
}

// One step of every partition + the exchanges.
// t_base != NULL: the step is being captured into a step graph whose first
// step is t0; its kernels read t0 from *t_base (StepArgs::t_base)
sim_status step_once(sim_s *h, const int32_t *t_base = nullptr, int t0 = 0) {
  const int t = h->t, W = h->world;
  cudaStream_t st = h->stream;
  auto step_args = [&](const Part &P, int tt) {
    StepArgs a = ::step_args(P, tt);
    if (t_base) {
      a.t = tt - t0;
      a.t_base = t_base;
    }
    return a;
  };
  for (Part &P : h->parts) {
    if (h->P.record_decisions) {
      CK(h, cudaMemsetAsync(P.A.r_ins, 0, h->nv, st));
      CK(h, cudaMemsetAsync(P.A.r_mark, 0, h->nv, st));
      CK(h, cudaMemsetAsync(P.A.r_leader, 0xff, h->nv * 4, st));
      CK(h, cudaMemsetAsync(P.A.r_lc, 0, h->nv, st));
    }
  }
  cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
  if (h->timing) {
    while (h->ev_pool.size() < h->ev_used + 3) {
      cudaEvent_t ev;
      CK(h, cudaEventCreate(&ev));
      h->ev_pool.push_back(ev);
    }
    for (int q = 0; q < 3; ++q) e[q] = h->ev_pool[h->ev_used + q];
    h->ev_used += 3;
    CK(h, cudaEventRecord(e[0], st));
  }
  // MAX_PRESSURE lane counts (L39): k_signal reads those of state(t), k_step
  // (and k_absorb) accumulate those of state(t+1), the buffer of t+2 is cleared
  int32_t *cnt_next = h->any_maxp ? h->lcnt[(t + 1) % 3] : nullptr;
  if (h->any_maxp) CK(h, cudaMemsetAsync(h->lcnt[(t + 2) % 3], 0, h->nl * 4, st));
  for (Part &P : h->parts) {
    SignalArgs sg = P.SG;
    sg.lane_cnt = h->lcnt[t % 3];
    sg.cnt_buf = t % 3;
    launch_signal(sg, st);
    h->n_launch += h->nj > 0;
  }
  if (h->timing) CK(h, cudaEventRecord(e[1], st));
  for (Part &P : h->parts) {
    StepArgs a = step_args(P, t);
    a.lane_cnt_next = cnt_next;
    launch_prep(a, st);
    launch_step(a, st, h->smem);
    h->n_launch += 2 * (a.n_own > 0);
  }
  if (h->timing) CK(h, cudaEventRecord(e[2], st));
  if (h->ipc) {                                     // direct transport: movers and summaries are
    sim_status bs = barrier(h);                     // already in the owners' buffers (NEXT-2)
    if (bs) return bs;
  }
  if (W > 1 && !h->direct) {
    // 1. migration: headers carry the counts, whole regions are exchanged
    for (Part &P : h->parts) { launch_mig_header(P.out_buf, P.A.out_off, P.A.out_cap, P.out_cnt, W, st); h->n_launch++; }
    if (h->loopback) {
      for (Part &P : h->parts)
        for (int q = 0; q < W; ++q)
          if (P.out_cap[q]) {
            Part &Q = h->parts[q];
            CK(h, cudaMemcpyAsync(Q.in_buf + Q.in_off[P.rank], P.out_buf + P.out_off[q],
                                  (P.out_cap[q] + 1) * sizeof(MigRec), cudaMemcpyDeviceToDevice, st));
          }
    } else {
      Part &P = h->parts[0];
      NK(h, g_nccl.GroupStart());
      for (int q = 0; q < W; ++q) {
        if (P.out_cap[q])
          NK(h, g_nccl.Send(P.out_buf + P.out_off[q], (P.out_cap[q] + 1) * sizeof(MigRec), kNcclInt8, q, h->comm, st));
        if (P.in_cap[q])
          NK(h, g_nccl.Recv(P.in_buf + P.in_off[q], (P.in_cap[q] + 1) * sizeof(MigRec), kNcclInt8, q, h->comm, st));
      }
      NK(h, g_nccl.GroupEnd());
    }
    for (Part &P : h->parts) {
      StepArgs a = step_args(P, t);
      a.lane_cnt_next = cnt_next;
      launch_absorb(a, P.in_buf, P.in_off_d, P.in_cap_d, W, st);
      h->n_launch++;
    }
    // every rank counted its own lanes (loopback partitions share one buffer)
    if (cnt_next && !h->loopback)
      NK(h, g_nccl.AllReduce(cnt_next, cnt_next, h->nl, 2 /*ncclInt32*/, kNcclSum, h->comm, st));
    // 2. halo: the first-vehicle summaries of the lanes each peer reads
    for (Part &P : h->parts) {
      StepArgs a = step_args(P, t);
      launch_halo_pack(a, P.hs_lanes, P.hs_buf, P.hs_n, st);
      h->n_launch++;
    }
    if (h->loopback) {
      for (Part &P : h->parts)
        for (int q = 0; q < W; ++q) {
          const int n = P.hs_off[q + 1] - P.hs_off[q];
          if (!n) continue;
          Part &Q = h->parts[q];
          CK(h, cudaMemcpyAsync(Q.hr_buf + Q.hr_off[P.rank], P.hs_buf + P.hs_off[q], n * sizeof(HaloRec),
                                cudaMemcpyDeviceToDevice, st));
        }
    } else {
      Part &P = h->parts[0];
      NK(h, g_nccl.GroupStart());
      for (int q = 0; q < W; ++q) {
        const int ns = P.hs_off[q + 1] - P.hs_off[q], nr = P.hr_off[q + 1] - P.hr_off[q];
        if (ns) NK(h, g_nccl.Send(P.hs_buf + P.hs_off[q], ns * sizeof(HaloRec), kNcclInt8, q, h->comm, st));
        if (nr) NK(h, g_nccl.Recv(P.hr_buf + P.hr_off[q], nr * sizeof(HaloRec), kNcclInt8, q, h->comm, st));
      }
      NK(h, g_nccl.GroupEnd());
    }
    for (Part &P : h->parts) {
      StepArgs a = step_args(P, t);
      launch_halo_unpack(a, P.hr_lanes, P.hr_buf, P.hr_n, st);
      h->n_launch++;
    }
  }
  h->t += 1;
  return SIM_OK;
}

// After a change of lane directions / restrictions / speeds: recompute the
// usable flags, reachable roads and tile descriptors and stream them.
sim_status push_lane_tables(sim_s *h) {
  sim_status st;
  compute_usable(h);
  // one staging buffer: the outroads table followed by the usable bytes
  std::vector<uint8_t> buf((size_t)h->nl + h->outroads.size() * 4);
  std::memcpy(buf.data(), h->outroads.data(), h->outroads.size() * 4);
  std::memcpy(buf.data() + h->outroads.size() * 4, h->usable.data(), h->nl);
  st = push_staging(h, buf.data(), buf.size(), h->stage_dir_d);
  if (st) return st;
  for (Part &P : h->parts) {
    CK(h, cudaMemcpyAsync(P.outroads_d, h->stage_dir_d, h->outroads.size() * 4,
                          cudaMemcpyDeviceToDevice, h->stream));
    CK(h, cudaMemcpyAsync(P.usable_d, h->stage_dir_d + h->outroads.size() * 4, h->nl,
                          cudaMemcpyDeviceToDevice, h->stream));
  }
  // tile descriptors carry usable flags and reachable roads: stream them too
  st = push_staging(h, h->desc.data(), h->desc.size() * 4, h->parts[0].desc_d);
  if (st) return st;
  for (size_t i = 1; i < h->parts.size(); ++i)
    CK(h, cudaMemcpyAsync(h->parts[i].desc_d, h->parts[0].desc_d, h->desc.size() * 4,
                          cudaMemcpyDeviceToDevice, h->stream));
  return SIM_OK;
}

// MAX_PRESSURE switched on by a setter: the lane counts of state(t) are
// rebuilt from the slabs + inboxes (k_lane_stats) and the other buffers cleared.
sim_status rebuild_counts(sim_s *h) {
  const int t = h->t;
  CK(h, cudaMemsetAsync(h->lcnt[t % 3], 0, h->nl * 4, h->stream));
  CK(h, cudaMemsetAsync(h->lcnt[(t + 1) % 3], 0, h->nl * 4, h->stream));
  CK(h, cudaMemsetAsync(h->lcnt[(t + 2) % 3], 0, h->nl * 4, h->stream));
  int32_t *wscratch = h->parts[0].lanestat_d + h->nl;
  for (Part &P : h->parts) {
    StepArgs a = step_args(P, t);
    launch_lane_stats(a, h->lcnt[t % 3], wscratch, nullptr, h->P.queue_zone_m, h->stream);
    h->n_launch += 1;
  }
  // (direct transport: each count stays with the lane's owner, k_signal reads it there)
  if (h->comm) NK(h, g_nccl.AllReduce(h->lcnt[t % 3], h->lcnt[t % 3], h->nl, 2 /*ncclInt32*/, kNcclSum, h->comm, h->stream));
  return SIM_OK;
}

// Per-junction requests (later entries for the same junction win):
// kind 0 phase (request), 1 policy (pol_request), 2 duration (dur_request);
// deduplicated on the host and applied by one thread per junction.
sim_status push_junction_requests(sim_s *h, int m, const int32_t *junctions, const int32_t *vals,
                                  int kind) {
  sim_status st;
  // fast path: strictly increasing junction ids (every junction once, e.g. a
  // whole-network controller) need no de-duplication and go straight to the
  // pinned staging buffer
  bool uniq = true;
  for (int i = 1; i < m && uniq; ++i) uniq = junctions[i - 1] < junctions[i];
  if (uniq) {
    if (h->stage_cap < 2 * m) {
      if (h->stage_d) { CK(h, cudaStreamSynchronize(h->stream)); cudaFree(h->stage_d); }
      CK(h, cudaMalloc(&h->stage_d, 2 * (size_t)m * 4));
      h->stage_cap = 2 * m;
    }
    const size_t bytes = 2 * (size_t)m * 4;
    if (h->pinned_cap < bytes) {
      if (h->pinned) { CK(h, cudaEventSynchronize(h->stage_ev)); cudaFreeHost(h->pinned); }
      h->pinned = nullptr;
      CK(h, cudaHostAlloc(&h->pinned, bytes, cudaHostAllocDefault));
      h->pinned_cap = bytes;
    } else {
      CK(h, cudaEventSynchronize(h->stage_ev));
    }
    std::memcpy(h->pinned, junctions, (size_t)m * 4);
    std::memcpy(reinterpret_cast<int32_t *>(h->pinned) + m, vals, (size_t)m * 4);
    CK(h, cudaMemcpyAsync(h->stage_d, h->pinned, bytes, cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaEventRecord(h->stage_ev, h->stream));
    for (Part &P : h->parts) {
      int32_t *dst = kind == 0 ? P.SG.request : (kind == 1 ? P.SG.pol_request : P.SG.dur_request);
      launch_apply_requests(dst, h->stage_d, h->stage_d + m, m, h->stream);
      h->n_launch++;
    }
    return SIM_OK;
  }
  h->req_mark.resize(h->nj, -1);
  std::vector<int32_t> buf(2 * (size_t)m);
  int u = 0;
  for (int i = m - 1; i >= 0; --i) {
    const int j = junctions[i];
    if (h->req_mark[j] == h->req_epoch) continue;
    h->req_mark[j] = h->req_epoch;
    buf[u] = j;
    buf[m + u] = vals[i];
    ++u;
  }
  if (++h->req_epoch == 0x7fffffff) { h->req_epoch = 0; std::fill(h->req_mark.begin(), h->req_mark.end(), -1); }
  std::memmove(buf.data() + u, buf.data() + m, u * 4);
  if (h->stage_cap < 2 * u) {
    if (h->stage_d) { CK(h, cudaStreamSynchronize(h->stream)); cudaFree(h->stage_d); }
    CK(h, cudaMalloc(&h->stage_d, 2 * (size_t)u * 4));
    h->stage_cap = 2 * u;
  }
  st = push_staging(h, buf.data(), 2 * (size_t)u * 4, h->stage_d);
  if (st) return st;
  for (Part &P : h->parts) {
    int32_t *dst = kind == 0 ? P.SG.request : (kind == 1 ? P.SG.pol_request : P.SG.dur_request);
    launch_apply_requests(dst, h->stage_d, h->stage_d + u, u, h->stream);
    h->n_launch++;
  }
  return SIM_OK;
}

}  // namespace

extern "C" {

static void destroy_impl(sim_s *h) {
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (size_t i = 0; i < h->allocs.size(); ++i) {
    if (!h->alloc_hooked[i]) cudaFree(h->allocs[i]);
    else if (h->P.free_) h->P.free_(h->allocs[i], h->P.alloc_ctx);
  }
  if (h->stage_d) cudaFree(h->stage_d);
  if (h->pinned) cudaFreeHost(h->pinned);
  if (h->rd_pinned) cudaFreeHost(h->rd_pinned);
  if (h->stage_ev) cudaEventDestroy(h->stage_ev);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  if (h->comm) g_nccl.CommDestroy(h->comm);
  for (void *q : h->ipc_opened) cudaIpcCloseMemHandle(q);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

sim_status sim_ipc_export(sim_handle h, uint8_t *out, int32_t cap, int32_t *n_bytes) {
  sim_status st = check(h);
  if (st) return st;
  if (!h->ipc) return fail(h, SIM_E_INVALID, "sim_ipc_export needs world > 1, direct = 1, loopback = 0");
  const int32_t need = kIpcBufs * (int32_t)(sizeof(cudaIpcMemHandle_t) + 1);
  if (n_bytes) *n_bytes = need;
  if (!out) return SIM_OK;                          // size query
  if (cap < need) return fail(h, SIM_E_INVALID, "export buffer too small");
  std::memset(out, 0, need);
  PeerView &V = h->parts[0].view;
  for (int k = 0; k < kIpcBufs; ++k) {
    void *ptr = *view_slot(V, k);
    if (!ptr) continue;                             // absent buffer (e.g. no groups): flag 0
    cudaIpcMemHandle_t mh;
    CK(h, cudaIpcGetMemHandle(&mh, ptr));
    std::memcpy(out + k * sizeof(cudaIpcMemHandle_t), &mh, sizeof(mh));
    out[kIpcBufs * sizeof(cudaIpcMemHandle_t) + k] = 1;
  }
  return SIM_OK;
}

sim_status sim_ipc_connect(sim_handle h, const uint8_t *blobs, int32_t n_bytes) {
  sim_status st = check(h);
  if (st) return st;
  if (!h->ipc) return fail(h, SIM_E_INVALID, "sim_ipc_connect needs world > 1, direct = 1, loopback = 0");
  if (h->connected) return fail(h, SIM_E_STATE, "already connected");
  const int32_t need = kIpcBufs * (int32_t)(sizeof(cudaIpcMemHandle_t) + 1);
  if (!blobs || n_bytes != need) return fail(h, SIM_E_INVALID, "blobs must be world x sim_ipc_export bytes");
  std::vector<PeerView> views(h->world);
  for (int q = 0; q < h->world; ++q) {
    if (q == h->rank) { views[q] = h->parts[0].view; continue; }
    const uint8_t *b = blobs + (size_t)q * need;
    PeerView V{};
    for (int k = 0; k < kIpcBufs; ++k) {
      if (!b[kIpcBufs * sizeof(cudaIpcMemHandle_t) + k]) continue;
      cudaIpcMemHandle_t mh;
      std::memcpy(&mh, b + k * sizeof(cudaIpcMemHandle_t), sizeof(mh));
      void *ptr = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&ptr, mh, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess)
        return fail(h, SIM_E_CUDA, std::string("cudaIpcOpenMemHandle (peer ") + std::to_string(q) +
                                       "): " + cudaGetErrorString(e));
      h->ipc_opened.push_back(ptr);
      *view_slot(V, k) = ptr;
    }
    views[q] = V;
  }
  st = upload_peers(h, views);
  if (st) return st;
  h->peer_views = views;
  h->connected = true;
  return SIM_OK;
}

sim_status sim_repartition(sim_handle h, const int32_t *road_owner, int32_t *moved_tiles) {
  sim_status st = check(h);
  if (st) return st;
  if (!h->direct) return fail(h, SIM_E_INVALID, "sim_repartition needs world > 1 and direct = 1");
  if (h->ipc && !h->connected) return fail(h, SIM_E_STATE, "direct transport: sim_ipc_connect has not been called");
  const int W = h->world, nt = h->nt, t = h->t;
  std::vector<int> own;
  if (road_owner) {
    own.assign(road_owner, road_owner + nt);
    for (int x : own)
      if (x < 0 || x >= W) return fail(h, SIM_E_RANGE, "road_owner out of [0, world)");
  } else {
    // balance the current load: vehicles per road tile (+1 so empty roads
    // still spread), summed over the partitions
    Part &P0 = h->parts[0];
    int32_t *d = P0.lanestat_d;
    std::vector<int64_t> w(nt, 1);
    std::vector<int32_t> c(nt);
    for (Part &P : h->parts) {
      int32_t *dst = h->loopback ? P.lanestat_d : d;
      CK(h, cudaMemsetAsync(dst, 0, nt * 4, h->stream));
      launch_tile_counts(step_args(P, t), dst, h->stream);
      h->n_launch++;
    }
    if (h->ipc) {
      st = allreduce_sum(h, 1, 1, 0, nt);
      if (st) return st;
    }
    for (Part &P : h->parts) {
      CK(h, cudaMemcpyAsync(c.data(), h->loopback ? P.lanestat_d : d, nt * 4, cudaMemcpyDeviceToHost, h->stream));
      st = device_check(h);
      if (st) return st;
      for (int T = 0; T < nt; ++T) w[T] += c[T];
      if (!h->loopback) break;
    }
    own = default_partition(h, W, &w);
  }
  int moved = 0;
  for (int T = 0; T < nt; ++T) moved += own[T] != h->tile_owner[T];
  if (moved_tiles) *moved_tiles = moved;
  if (!moved) return SIM_OK;
  st = barrier(h);                                  // every rank is at the same step boundary
  if (st) return st;
  if (!h->repart_own_d) {                           // allocated once, reused by later calls
    st = dalloc(h, &h->repart_own_d, (size_t)nt);
    if (st) return st;
  }
  int32_t *own_d = h->repart_own_d;
  CK(h, cudaMemcpyAsync(own_d, own.data(), nt * 4, cudaMemcpyHostToDevice, h->stream));
  for (Part &P : h->parts) {
    launch_rehome(step_args(P, t), own_d, h->stream);
    h->n_launch++;
  }
  st = barrier(h);                                  // the hand-over has landed everywhere
  if (st) return st;
  h->tile_owner = own;
  for (Part &P : h->parts) {
    P.tiles.clear();
    for (int T = 0; T < nt; ++T) if (own[T] == P.rank) P.tiles.push_back(T);
    std::vector<int> order(P.tiles);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return h->tile_cap[a] > h->tile_cap[b]; });
    if (!P.tiles_cap_d) {                           // own-tile list with room for every tile
      st = dalloc(h, &P.tiles_cap_d, (size_t)nt);
      if (st) return st;
    }
    int32_t *tl = P.tiles_cap_d;
    if (!order.empty())
      CK(h, cudaMemcpyAsync(tl, order.data(), order.size() * 4, cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaMemcpyAsync(const_cast<int32_t *>(P.A.tile_owner), own_d, nt * 4,
                          cudaMemcpyDeviceToDevice, h->stream));
    P.A.tiles = tl;
    P.A.n_own = (int)order.size();
  }
  return device_check(h);                           // host vectors above stay valid until done
}

sim_status sim_get_nccl_unique_id(uint8_t out[128]) {
  std::string err;
  if (!g_nccl.load(err)) return fail(nullptr, SIM_E_NCCL, err);
  NcclId id;
  int r = g_nccl.GetUniqueId(&id);
  if (r) return fail(nullptr, SIM_E_NCCL, std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(r));
  std::memcpy(out, id.internal, 128);
  return SIM_OK;
}

sim_status sim_create(const sim_graph *g, const sim_trips *tr, const sim_params *p,
                      sim_handle *out) {
  if (!out) return fail(nullptr, SIM_E_INVALID, "out is NULL");
  *out = nullptr;
  sim_s *h = new sim_s();
  sim_status st = validate_and_copy(h, g, tr, p);
  if (!st) st = build_tiles(h);
  if (!st) {
    h->world = std::max(1, p->world);
    h->rank = p->rank;
    h->loopback = h->world > 1 && p->loopback;
    h->direct = h->world > 1 && p->direct;
    h->ipc = h->direct && !h->loopback;
    if (h->world > 1 && !h->loopback && !h->direct &&
        (!p->nccl_id || p->rank < 0 || p->rank >= h->world))
      st = fail(h, SIM_E_INVALID, "world > 1 needs loopback = 1, direct = 1 or (nccl_id, 0 <= rank < world)");
    if (h->ipc && (p->rank < 0 || p->rank >= h->world || h->world > 32))
      st = fail(h, SIM_E_INVALID, "direct transport across processes needs 0 <= rank < world <= 32");
    if (h->world > 1 && h->nt < h->world) st = fail(h, SIM_E_INVALID, "fewer road tiles than partitions");
  }
  if (!st) {
    if (p->road_owner) {
      h->tile_owner.assign(p->road_owner, p->road_owner + h->nr);
      for (int x : h->tile_owner)
        if (x < 0 || x >= h->world) { st = fail(h, SIM_E_INVALID, "road_owner out of [0, world)"); break; }
    } else {
      h->tile_owner = h->world > 1 ? default_partition(h, h->world) : std::vector<int>(h->nr, 0);
    }
  }
  if (st) { g_create_err = h->err; delete h; return st; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    delete h;
    return fail(nullptr, SIM_E_CUDA, "no CUDA device available (the library has no CPU fallback)");
  }
  h->device = p->device;
  if (cudaSetDevice(h->device) != cudaSuccess) { delete h; return fail(nullptr, SIM_E_CUDA, "cudaSetDevice failed"); }
  if (p->stream) h->stream = (cudaStream_t)p->stream;
  else {
    cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    h->own_stream = true;
  }
  h->smem = step_smem_bytes();
  compute_usable(h);                 // usable flags, reachable roads, tile descriptors
  Plan plan;
  if (h->world > 1 && !h->direct) plan = make_plan(h);
  const int nparts = h->loopback ? h->world : 1;
  h->parts.resize(nparts);
  for (int i = 0; i < nparts && !st; ++i) {
    Part &P = h->parts[i];
    P.rank = h->loopback ? i : (h->world > 1 ? h->rank : 0);
    for (int T = 0; T < h->nt; ++T) if (h->tile_owner[T] == P.rank) P.tiles.push_back(T);
    st = alloc_part(h, P, (h->world > 1 && !h->direct) ? &plan : nullptr);
  }
  if (!st && h->direct) st = setup_direct(h);
  if (!st && h->world > 1 && !h->loopback && !h->direct) {
    std::string err;
    if (!g_nccl.load(err)) st = fail(h, SIM_E_NCCL, err);
    else {
      NcclId id;
      std::memcpy(id.internal, p->nccl_id, 128);
      int r = g_nccl.CommInitRank(&h->comm, h->world, id, h->rank);
      if (r) st = fail(h, SIM_E_NCCL, std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r));
    }
  }
  if (!st) {
    cudaError_t e = cudaMalloc(&h->stage_dir_d, 17 * (size_t)h->nl);
    if (e != cudaSuccess) st = fail(h, SIM_E_OOM, "cudaMalloc staging");
    else { h->allocs.push_back(h->stage_dir_d); h->alloc_hooked.push_back(0); }
  }
  if (!st) {
    if (cudaEventCreateWithFlags(&h->stage_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(h->stage_ev, h->stream) != cudaSuccess)
      st = fail(h, SIM_E_CUDA, "event creation failed");
  }
  if (!st) {
    HostState S;
    S.t = 0;
    const int nv = h->nv;
    S.status.assign(nv, ST_PENDING); S.lane.assign(nv, -1); S.cursor.assign(nv, 0);
    S.wait.assign(nv, 0); S.insert_time.assign(nv, -1); S.arrive_time.assign(nv, -1);
    S.s.assign(nv, 0.f); S.v.assign(nv, 0.f);
    for (int k = 0; k < nv; ++k)
      if (h->on0[k]) {
        S.status[k] = ST_DRIVING; S.lane[k] = h->start_lane[k]; S.s[k] = h->start_s[k];
        S.v[k] = h->start_v[k]; S.insert_time[k] = 0;
      }
    init_junctions(h, S);
    S.dir = h->dir;
    st = upload_state(h, S);
  }
  if (st) {
    g_create_err = h->err;
    destroy_impl(h);
    return st;
  }
  {
    std::lock_guard<std::mutex> lk(g_live_mu);
    g_live.insert(h);
  }
  *out = h;
  return SIM_OK;
}

// Step graphs: kGraphSteps steps captured once into a CUDA
// graph (k_signal -> k_prep -> k_step per step, chained by programmatic
// dependent launches) and replayed, so a long sim_step(n) costs one launch per
// kGraphSteps steps instead of three per step.  kGraphSteps = 6 is the period
// of the double- and triple-buffered step buffers, so the baked buffer
// pointers are those of the replay's steps whenever it starts at the same
// t mod 6; the absolute t comes from t_dev.  The graph is re-captured when any
// host-side launch argument changed since the capture (fingerprint below).
constexpr int kGraphSteps = 6;

void step_fingerprint(sim_s *h, std::vector<unsigned char> &fp) {
  fp.clear();
  auto put = [&](const void *p, size_t n) {
    const unsigned char *c = reinterpret_cast<const unsigned char *>(p);
    fp.insert(fp.end(), c, c + n);
  };
  const int hdr[8] = {h->t % kGraphSteps, h->P.record_decisions, h->any_maxp ? 1 : 0, h->world,
                      h->direct ? 1 : 0, h->loopback ? 1 : 0, h->smem, (int)h->parts.size()};
  put(hdr, sizeof hdr);
  for (const Part &P : h->parts) {
    put(&P.A, sizeof(StepArgs));
    put(&P.SG, sizeof(SignalArgs));
  }
}

bool graphs_usable(sim_s *h) {
  // not with the per-step host-side barrier (IPC) or NCCL calls, nor while
  // per-kernel timing events are recorded
  return !h->P.no_step_graphs && !h->g_off && !h->timing && !h->ipc && !h->comm;
}

// the graph for the current t mod 6 and host state; false: use eager steps
sim_status ensure_graph(sim_s *h, bool *ok) {
  *ok = false;
  std::vector<unsigned char> fp;
  step_fingerprint(h, fp);
  if (h->gexec && fp == h->g_fp) { *ok = true; return SIM_OK; }
  if (h->gexec) {
    CK(h, cudaGraphExecDestroy(h->gexec));
    h->gexec = nullptr;
  }
  if (!h->t_dev) {
    sim_status s = dalloc(h, &h->t_dev, 1);
    if (s) return s;
  }
  init_step_launch(h->smem);
  if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();                             // e.g. the legacy default stream: stay eager
    h->g_off = true;
    return SIM_OK;
  }
  const int t0 = h->t;
  const int64_t nl0 = h->n_launch;
  sim_status s = SIM_OK;
  for (int k = 0; k < kGraphSteps && s == SIM_OK; ++k) s = step_once(h, h->t_dev, t0);
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(h->stream, &g);
  h->t = t0;
  const int64_t per = h->n_launch - nl0;
  h->n_launch = nl0;
  if (s != SIM_OK || e != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    if (s != SIM_OK) return s;
    h->sticky = SIM_E_CUDA;
    return fail(h, SIM_E_CUDA, std::string("step graph capture: ") + cudaGetErrorString(e));
  }
  const cudaError_t ei = cudaGraphInstantiate(&h->gexec, g, 0);
  cudaGraphDestroy(g);
  if (ei != cudaSuccess) {
    h->gexec = nullptr;
    h->sticky = SIM_E_CUDA;
    return fail(h, SIM_E_CUDA, std::string("step graph instantiate: ") + cudaGetErrorString(ei));
  }
  h->g_fp.swap(fp);
  h->g_launches = per;
  *ok = true;
  return SIM_OK;
}

sim_status sim_step(sim_handle h, int32_t n) {
  sim_status st = check(h);
  if (st) return st;
  if (n < 0) return fail(h, SIM_E_RANGE, "n must be >= 0");
  if (n > 0 && h->ipc) {                            // host-side changes of every rank precede
    st = barrier(h);                                // the first peer write of this call
    if (st) return st;
  }
  int i = 0;
  if (n >= 2 * kGraphSteps && graphs_usable(h)) {
    bool ok = false;
    st = ensure_graph(h, &ok);
    if (st) return st;
    for (; ok && n - i >= kGraphSteps; i += kGraphSteps) {
      launch_set_i32(h->t_dev, h->t, h->stream);
      CK(h, cudaGraphLaunch(h->gexec, h->stream));
      h->t += kGraphSteps;
      h->n_launch += h->g_launches + 1;
    }
  }
  for (; i < n; ++i) {
    st = step_once(h);
    if (st) return st;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    h->sticky = SIM_E_CUDA;
    return fail(h, SIM_E_CUDA, std::string("launch: ") + cudaGetErrorString(e));
  }
  return SIM_OK;
}

sim_status sim_sync(sim_handle h) {
  sim_status st = check(h);
  if (st) return st;
  return device_check(h);
}

sim_status sim_set_signal_phase_batch(sim_handle h, int32_t m, const int32_t *junctions,
                                      const int32_t *phases) {
  sim_status st = check(h);
  if (st) return st;
  if (m < 0 || (m > 0 && (!junctions || !phases))) return fail(h, SIM_E_INVALID, "bad batch");
  for (int i = 0; i < m; ++i) {
    int j = junctions[i];
    if (j < 0 || j >= h->nj) return fail(h, SIM_E_RANGE, "junction out of range");
    int K = h->ph_off[j + 1] - h->ph_off[j];
    if (phases[i] < 0 || phases[i] >= K) return fail(h, SIM_E_RANGE, "phase out of range");
  }
  if (m == 0) return SIM_OK;
  return push_junction_requests(h, m, junctions, phases, 0);   // replicated controllers
}

sim_status sim_set_signal_phase(sim_handle h, int32_t j, int32_t p) {
  return sim_set_signal_phase_batch(h, 1, &j, &p);
}

sim_status sim_set_lane_direction_batch(sim_handle h, int32_t m, const int32_t *lanes,
                                        const int32_t *dirs) {
  sim_status st = check(h);
  if (st) return st;
  if (m < 0 || (m > 0 && (!lanes || !dirs))) return fail(h, SIM_E_INVALID, "bad batch");
  for (int i = 0; i < m; ++i) {
    if (lanes[i] < 0 || lanes[i] >= h->nl || dirs[i] < 0 || dirs[i] > 1)
      return fail(h, SIM_E_RANGE, "lane or direction out of range");
    int k = h->kind[lanes[i]];
    if (k != KIND_DYNAMIC && k != KIND_TIDAL)
      return fail(h, SIM_E_INVALID, "lane " + std::to_string(lanes[i]) + " is neither DYNAMIC nor TIDAL");
  }
  for (int i = 0; i < m; ++i) {
    int l = lanes[i];
    h->dir[l] = (uint8_t)dirs[i];
    if (h->kind[l] == KIND_TIDAL && h->partner[l] >= 0) h->dir[h->partner[l]] = (uint8_t)(1 - dirs[i]);
  }
  if (m == 0) return SIM_OK;
  return push_lane_tables(h);
}

sim_status sim_set_lane_direction(sim_handle h, int32_t lane, int32_t dir) {
  return sim_set_lane_direction_batch(h, 1, &lane, &dir);
}

sim_status sim_set_signal_policy_batch(sim_handle h, int32_t m, const int32_t *junctions,
                                       const int32_t *policies) {
  sim_status st = check(h);
  if (st) return st;
  if (m < 0 || (m > 0 && (!junctions || !policies))) return fail(h, SIM_E_INVALID, "bad batch");
  for (int i = 0; i < m; ++i) {
    if (junctions[i] < 0 || junctions[i] >= h->nj) return fail(h, SIM_E_RANGE, "junction out of range");
    if (policies[i] < POL_NONE || policies[i] > POL_MAXP) return fail(h, SIM_E_RANGE, "policy out of range");
  }
  if (m == 0) return SIM_OK;
  bool maxp = false;
  for (int i = 0; i < m; ++i) maxp |= policies[i] == POL_MAXP;
  if (maxp && !h->any_maxp) {                        // counts of state(t) needed from the next step
    h->any_maxp = true;
    st = rebuild_counts(h);
    if (st) return st;
  }
  return push_junction_requests(h, m, junctions, policies, 1);
}

sim_status sim_set_signal_duration_batch(sim_handle h, int32_t m, const int32_t *junctions,
                                         const int32_t *steps) {
  sim_status st = check(h);
  if (st) return st;
  if (m < 0 || (m > 0 && (!junctions || !steps))) return fail(h, SIM_E_INVALID, "bad batch");
  for (int i = 0; i < m; ++i) {
    if (junctions[i] < 0 || junctions[i] >= h->nj) return fail(h, SIM_E_RANGE, "junction out of range");
    if (steps[i] < 1) return fail(h, SIM_E_RANGE, "duration must be >= 1 step");
  }
  if (m == 0) return SIM_OK;
  return push_junction_requests(h, m, junctions, steps, 2);
}

sim_status sim_set_signal_duration(sim_handle h, int32_t j, int32_t steps) {
  return sim_set_signal_duration_batch(h, 1, &j, &steps);
}

sim_status sim_set_signal_policy(sim_handle h, int32_t j, int32_t policy) {
  return sim_set_signal_policy_batch(h, 1, &j, &policy);
}

sim_status sim_set_lane_max_speed_batch(sim_handle h, int32_t m, const int32_t *lanes,
                                        const float *speeds) {
  sim_status st = check(h);
  if (st) return st;
  if (m < 0 || (m > 0 && (!lanes || !speeds))) return fail(h, SIM_E_INVALID, "bad batch");
  for (int i = 0; i < m; ++i) {
    if (lanes[i] < 0 || lanes[i] >= h->nl) return fail(h, SIM_E_RANGE, "lane out of range");
    if (!(speeds[i] > 0.0f) || !std::isfinite(speeds[i])) return fail(h, SIM_E_RANGE, "max speed must be > 0");
  }
  if (m == 0) return SIM_OK;
  for (int i = 0; i < m; ++i) h->vmax[lanes[i]] = speeds[i];
  st = push_staging(h, h->vmax.data(), h->vmax.size() * 4, h->parts[0].lane_vmax_d);
  if (st) return st;
  for (size_t i = 1; i < h->parts.size(); ++i)
    CK(h, cudaMemcpyAsync(h->parts[i].lane_vmax_d, h->parts[0].lane_vmax_d, h->vmax.size() * 4,
                          cudaMemcpyDeviceToDevice, h->stream));
  return push_lane_tables(h);                        // descriptors carry the lane speeds
}

sim_status sim_set_lane_max_speed(sim_handle h, int32_t lane, float v) {
  return sim_set_lane_max_speed_batch(h, 1, &lane, &v);
}

sim_status sim_set_lane_restriction_batch(sim_handle h, int32_t m, const int32_t *lanes,
                                          const int32_t *flags) {
  sim_status st = check(h);
  if (st) return st;
  if (m < 0 || (m > 0 && (!lanes || !flags))) return fail(h, SIM_E_INVALID, "bad batch");
  for (int i = 0; i < m; ++i)
    if (lanes[i] < 0 || lanes[i] >= h->nl || flags[i] < 0 || flags[i] > 1)
      return fail(h, SIM_E_RANGE, "lane or flag out of range");
  if (m == 0) return SIM_OK;
  if (h->restricted.size() != (size_t)h->nl) h->restricted.assign(h->nl, 0);
  for (int i = 0; i < m; ++i) h->restricted[lanes[i]] = (uint8_t)flags[i];
  return push_lane_tables(h);
}

sim_status sim_set_lane_restriction(sim_handle h, int32_t lane, int32_t flag) {
  return sim_set_lane_restriction_batch(h, 1, &lane, &flag);
}

sim_status sim_set_vehicle_route_batch(sim_handle h, int32_t m, const int32_t *vids,
                                       const int32_t *route_offsets, const int32_t *roads,
                                       const float *end_s) {
  sim_status st = check(h);
  if (st) return st;
  if (m < 0 || (m > 0 && (!vids || !route_offsets || !roads || !end_s)))
    return fail(h, SIM_E_INVALID, "bad batch");
  if (m == 0) return SIM_OK;
  if (route_offsets[0] != 0) return fail(h, SIM_E_INVALID, "route_offsets[0] != 0");
  std::vector<int> last(m, 1);                       // later entries for a vehicle win
  {
    std::vector<int> seen;
    for (int i = m - 1; i >= 0; --i) {
      if (vids[i] < 0 || vids[i] >= h->nv) return fail(h, SIM_E_RANGE, "vehicle out of range");
      if (std::find(seen.begin(), seen.end(), vids[i]) != seen.end()) last[i] = 0;
      else seen.push_back(vids[i]);
    }
  }
  for (int i = 0; i < m; ++i) {
    const int a = route_offsets[i], b = route_offsets[i + 1];
    if (b <= a || b - a > 65000) return fail(h, SIM_E_INVALID, "route length must be in [1, 65000]");
    for (int e = a; e < b; ++e) {
      if (roads[e] < 0 || roads[e] >= h->nr) return fail(h, SIM_E_RANGE, "route road out of range");
      if (e + 1 < b && !std::binary_search(h->radj[roads[e]].begin(), h->radj[roads[e]].end(), roads[e + 1]))
        return fail(h, SIM_E_INVALID, "consecutive route roads are not connected");
    }
    const int dl = h->road_lanes[h->road_off[roads[b - 1]]];
    if (!(end_s[i] >= 0 && end_s[i] <= h->L[dl])) return fail(h, SIM_E_INVALID, "end_s outside [0, L]");
  }
  std::vector<int32_t> sel;                          // batch entries kept
  for (int i = 0; i < m; ++i) if (last[i]) sel.push_back(i);
  const int u = (int)sel.size();
  st = device_check(h);
  if (st) return st;
  // where is each vehicle (cursor, lane) and what is its status
  std::vector<int32_t> hv(u), hb(u);
  for (int q = 0; q < u; ++q) { hv[q] = vids[sel[q]]; hb[q] = q; }
  int32_t *d = nullptr;
  uint8_t *dst8 = nullptr;
  CK(h, cudaMalloc(&d, (4 * (size_t)u + 8) * 4));
  CK(h, cudaMalloc(&dst8, (size_t)u * h->parts.size() + 8));
  int32_t *d_vid = d, *d_idx = d + u, *d_out = d + 2 * u;
  CK(h, cudaMemcpy(d_vid, hv.data(), u * 4, cudaMemcpyHostToDevice));
  CK(h, cudaMemcpy(d_idx, hb.data(), u * 4, cudaMemcpyHostToDevice));
  CK(h, dmemset(h, d_out, 0xff, 2 * (size_t)u * 4));
  for (size_t pi = 0; pi < h->parts.size(); ++pi) {
    Part &P = h->parts[pi];
    StepArgs a = step_args(P, h->t);
    launch_scatter_i32(P.patch_d, d_vid, d_idx, 0, u, h->stream);
    launch_locate(a, P.patch_d, d_out, h->stream);
    launch_scatter_i32(P.patch_d, d_vid, nullptr, -1, u, h->stream);
    launch_gather_u8(P.A.status, d_vid, dst8 + pi * u, u, h->stream);
  }
  std::vector<int32_t> loc(2 * (size_t)u);
  std::vector<uint8_t> stt((size_t)u * h->parts.size());
  CK(h, cudaMemcpyAsync(loc.data(), d_out, 2 * (size_t)u * 4, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaMemcpyAsync(stt.data(), dst8, stt.size(), cudaMemcpyDeviceToHost, h->stream));
  st = device_check(h);
  cudaFree(d_vid);
  cudaFree(dst8);
  if (st) return st;
  if (h->comm || h->ipc) {
    // one process per rank: a vehicle is located by the rank that owns its
    // tile and may have finished on any rank — sum (position + 1, finished)
    // over the ranks so that every rank validates and applies identically
    std::vector<int32_t> x(3 * (size_t)u, 0);
    for (int q = 0; q < u; ++q) {
      if (loc[2 * q] >= 0) { x[2 * q] = loc[2 * q] + 1; x[2 * q + 1] = loc[2 * q + 1] + 1; }
      x[2 * (size_t)u + q] = stt[q] == ST_FINISHED;
    }
    Part &P0 = h->parts[0];
    CK(h, cudaMemcpyAsync(P0.xch_d, x.data(), x.size() * 4, cudaMemcpyHostToDevice, h->stream));
    st = allreduce_sum(h, 3, 1, 0, 3 * (int64_t)u);
    if (st) return st;
    CK(h, cudaMemcpyAsync(x.data(), P0.xch_d, x.size() * 4, cudaMemcpyDeviceToHost, h->stream));
    st = device_check(h);
    if (st) return st;
    for (int q = 0; q < u; ++q) {
      loc[2 * q] = x[2 * q] - 1;
      loc[2 * q + 1] = x[2 * q + 1] - 1;
      stt[q] = x[2 * (size_t)u + q] ? ST_FINISHED : ST_PENDING;
    }
  }
  // validation against the current position (L46); nothing changes on failure
  std::vector<int32_t> drv;                          // DRIVING vehicles of the batch
  for (int q = 0; q < u; ++q) {
    const int i = sel[q], k = vids[i];
    const int *r = roads + route_offsets[i];
    const int n = route_offsets[i + 1] - route_offsets[i];
    const int c = loc[2 * q], lane = loc[2 * q + 1];
    bool fin = false;
    for (size_t pi = 0; pi < h->parts.size(); ++pi) fin |= stt[pi * u + q] == ST_FINISHED;
    const std::string id = " (vehicle " + std::to_string(k) + ")";
    if (c >= 0) {                                    // DRIVING
      if (r[0] != route_at(h, k, c)) return fail(h, SIM_E_INVALID, "new route must start with the vehicle's current road" + id);
      if (!is_road(h, lane) && (n < 2 || r[1] != route_at(h, k, c + 1)))
        return fail(h, SIM_E_INVALID, "inside a junction the route must continue with the committed road" + id);
      drv.push_back(k);
    } else if (fin) {
      return fail(h, SIM_E_INVALID, "vehicle already finished" + id);
    } else {                                         // PENDING: start lane stays
      if (r[0] != route_at(h, k, 0)) return fail(h, SIM_E_INVALID, "new route must start with the trip's first road" + id);
    }
  }
  // apply: append the routes, point the vehicles at them
  const size_t old_n = h->route.size();
  std::vector<int32_t> ns(u), nl(u);
  std::vector<float> ne(u);
  for (int q = 0; q < u; ++q) {
    const int i = sel[q], k = vids[i];
    const int n = route_offsets[i + 1] - route_offsets[i];
    ns[q] = (int32_t)h->route.size();
    nl[q] = n;
    ne[q] = end_s[i];
    h->route.insert(h->route.end(), roads + route_offsets[i], roads + route_offsets[i + 1]);
    h->rstart[k] = ns[q];
    h->rlen[k] = n;
    h->end_s[k] = end_s[i];
  }
  if ((int64_t)h->route.size() > 2000000000LL) return fail(h, SIM_E_INVALID, "route storage exceeds 32-bit offsets");
  const bool grow = (int64_t)h->route.size() > h->route_cap;
  if (grow) h->route_cap = (int64_t)h->route.size() * 2;
  for (Part &P : h->parts) {
    if (grow) {                                      // the old buffer is released at destroy
      st = dalloc(h, &P.route_d, (size_t)h->route_cap);
      if (st) return st;
      P.A.route = P.route_d;
      CK(h, cudaMemcpy(P.route_d, h->route.data(), h->route.size() * 4, cudaMemcpyHostToDevice));
    } else {
      CK(h, cudaMemcpy(P.route_d + old_n, h->route.data() + old_n, (h->route.size() - old_n) * 4,
                       cudaMemcpyHostToDevice));
    }
  }
  int32_t *e = nullptr;
  CK(h, cudaMalloc(&e, (4 * (size_t)u + drv.size() + 8) * 4));
  CK(h, cudaMemcpy(e, hv.data(), u * 4, cudaMemcpyHostToDevice));
  CK(h, cudaMemcpy(e + u, ns.data(), u * 4, cudaMemcpyHostToDevice));
  CK(h, cudaMemcpy(e + 2 * u, nl.data(), u * 4, cudaMemcpyHostToDevice));
  CK(h, cudaMemcpy(e + 3 * u, ne.data(), u * 4, cudaMemcpyHostToDevice));
  if (!drv.empty()) CK(h, cudaMemcpy(e + 4 * u, drv.data(), drv.size() * 4, cudaMemcpyHostToDevice));
  for (Part &P : h->parts) {
    launch_scatter_i32(P.route_start_d, e, e + u, 0, u, h->stream);
    launch_scatter_i32(P.route_len_d, e, e + 2 * u, 0, u, h->stream);
    launch_scatter_f32(P.end_s_d, e, reinterpret_cast<const float *>(e + 3 * u), u, h->stream);
    if (!drv.empty()) {                              // restart at cursor 0 of the new route
      StepArgs a = step_args(P, h->t);
      a.route = P.route_d;
      launch_scatter_i32(P.patch_d, e + 4 * u, nullptr, 0, (int)drv.size(), h->stream);
      launch_patch_routes(a, P.patch_d, h->stream);
      launch_scatter_i32(P.patch_d, e + 4 * u, nullptr, -1, (int)drv.size(), h->stream);
    }
    h->n_launch += 6;
  }
  st = device_check(h);
  cudaFree(e);
  return st;
}

sim_status sim_set_vehicle_route(sim_handle h, int32_t vid, int32_t n, const int32_t *roads,
                                 float end_s) {
  const int32_t off[2] = {0, n};
  return sim_set_vehicle_route_batch(h, 1, &vid, off, roads, &end_s);
}

sim_status sim_query_sizes(sim_handle h, sim_sizes *out) {
  if (!h || !is_live(h)) return SIM_E_STATE;
  if (!out) return SIM_E_INVALID;
  out->n_vehicles = h->nv; out->n_lanes = h->nl; out->n_junctions = h->nj; out->n_tiles = h->nt;
  out->device_bytes = h->bytes;
  return SIM_OK;
}

// Vehicles on the tiles of the handle's partition(s) are read from the slabs /
// inboxes; cold fields are merged over partitions (a vehicle's FINISHED record
// lives on the partition where it arrived).
// sim_read_state / sim_read_state_global: the vehicles of every partition
// this process can see — its own (loopback: all of them), or with `global`
// and the direct transport across processes every rank's, read through the
// peer mappings after the collective counter reduction.
static sim_status read_state_impl(sim_s *h, sim_state *o, bool global) {
  sim_status st = check(h);
  if (st) return st;
  if (!o) return fail(h, SIM_E_INVALID, "out is NULL");
  std::vector<long long> cs;
  st = read_counters(h, cs);                        // (collective across ranks: also the barrier)
  if (st) return st;
  const int par = h->t & 1, nv = h->nv, nt = h->nt;
  std::vector<int> lane(nv, -1), cur(nv, 0), wait(nv, 0), ins(nv, -1), arr(nv, -1);
  std::vector<float> vs(nv, 0.f), vv(nv, 0.f);
  std::vector<uint8_t> status(nv, ST_PENDING);
  std::vector<char> driving(nv, 0);
  struct Src { PeerView V; std::vector<int> tiles; };
  std::vector<Src> src;
  if (global && h->ipc) {
    for (int q = 0; q < h->world; ++q) {
      Src x;
      x.V = h->peer_views[q];
      for (int T = 0; T < nt; ++T) if (h->tile_owner[T] == q) x.tiles.push_back(T);
      src.push_back(std::move(x));
    }
  } else {
    for (Part &P : h->parts) src.push_back(Src{P.view, P.tiles});
  }
  for (Src &P : src) {
    std::vector<int> cnt(nt), icnt(nt);
    CK(h, cudaMemcpy(cnt.data(), P.V.cnt[par], nt * 4, cudaMemcpyDeviceToHost));
    CK(h, cudaMemcpy(icnt.data(), P.V.icnt[par], nt * 4, cudaMemcpyDeviceToHost));
    std::vector<InboxRec> ib(h->n_slots);
    CK(h, cudaMemcpy(ib.data(), P.V.inbox[par], ib.size() * sizeof(InboxRec), cudaMemcpyDeviceToHost));
    std::vector<uint8_t> pst(nv);
    std::vector<int> pins(nv), parr(nv), pwf(nv);
    CK(h, cudaMemcpy(pst.data(), P.V.status, nv, cudaMemcpyDeviceToHost));
    CK(h, cudaMemcpy(pins.data(), P.V.insert_time, nv * 4, cudaMemcpyDeviceToHost));
    CK(h, cudaMemcpy(parr.data(), P.V.arrive_time, nv * 4, cudaMemcpyDeviceToHost));
    CK(h, cudaMemcpy(pwf.data(), P.V.wait_fin, nv * 4, cudaMemcpyDeviceToHost));
    for (int k = 0; k < nv; ++k) {
      ins[k] = std::max(ins[k], pins[k]);
      if (pst[k] == ST_FINISHED) { status[k] = ST_FINISHED; arr[k] = parr[k]; wait[k] = pwf[k]; }
    }
    auto put = [&](int T, int k, float ss, float v_, uint32_t m, int w) {
      lane[k] = h->tile_lanes[h->tile_lane_off[T] + (m & 0xff)];
      vs[k] = ss; vv[k] = v_; cur[k] = (int)(m >> 16); wait[k] = w; driving[k] = 1;
    };
    for (int T : P.tiles) {
      for (int i = 0; i < cnt[T]; ++i) {
        const InboxRec &r = ib[h->tile_base[T] + h->tile_cap[T] - cnt[T] + i];
        put(T, r.vid, r.s, r.v, r.meta, r.wait);
      }
      for (int i = 0; i < icnt[T]; ++i) { const InboxRec &r = ib[h->tile_ibase[T] + i]; put(T, r.vid, r.s, r.v, r.meta, r.wait); }
    }
  }
  for (int k = 0; k < nv; ++k) if (driving[k]) status[k] = ST_DRIVING;
  o->t = h->t;
  if (o->status) std::memcpy(o->status, status.data(), nv);
  for (int k = 0; k < nv; ++k) {
    bool d = status[k] == ST_DRIVING;
    if (o->lane) o->lane[k] = d ? lane[k] : -1;
    if (o->cursor) o->cursor[k] = d ? cur[k] : 0;
    if (o->wait_steps) o->wait_steps[k] = status[k] == ST_PENDING ? 0 : wait[k];
    if (o->insert_time) o->insert_time[k] = ins[k];
    if (o->arrive_time) o->arrive_time[k] = arr[k];
    if (o->s) o->s[k] = d ? vs[k] : 0.f;
    if (o->v) o->v[k] = d ? vv[k] : 0.f;
  }
  Part &P0 = h->parts[0];
  if (h->nj) {
    if (o->junc_policy) CK(h, cudaMemcpy(o->junc_policy, P0.SG.policy, h->nj, cudaMemcpyDeviceToHost));
    if (o->junc_phase) CK(h, cudaMemcpy(o->junc_phase, P0.SG.phase, h->nj * 4, cudaMemcpyDeviceToHost));
    if (o->junc_elapsed) CK(h, cudaMemcpy(o->junc_elapsed, P0.SG.elapsed, h->nj * 4, cudaMemcpyDeviceToHost));
    if (o->junc_yellow_left) CK(h, cudaMemcpy(o->junc_yellow_left, P0.SG.yellow_left, h->nj * 4, cudaMemcpyDeviceToHost));
    if (o->junc_pending) CK(h, cudaMemcpy(o->junc_pending, P0.SG.pending, h->nj * 4, cudaMemcpyDeviceToHost));
    if (o->junc_remaining) CK(h, cudaMemcpy(o->junc_remaining, P0.SG.remaining, h->nj * 4, cudaMemcpyDeviceToHost));
  }
  if (o->lane_dir) std::memcpy(o->lane_dir, h->dir.data(), h->nl);
  if (o->lane_signal) CK(h, cudaMemcpy(o->lane_signal, P0.A.lane_sig, h->nl, cudaMemcpyDeviceToHost));
  if (o->lane_offsets && o->lane_order) {
    std::vector<std::vector<int>> per(h->nl);
    if (!(global && h->ipc)) {
      // the order the step kernel itself merges (k_lane_order: stayers in
      // their record order + the inbox placed by rank), per partition
      std::vector<int32_t> ov(h->n_slots);
      std::vector<uint8_t> ol(h->n_slots);
      for (Part &P : h->parts) {
        if (!P.lo_vid_d) {
          sim_status sa = dalloc(h, &P.lo_vid_d, (size_t)h->n_slots);
          if (!sa) sa = dalloc(h, &P.lo_lane_d, (size_t)h->n_slots);
          if (sa) return sa;
        }
        launch_lane_order(step_args(P, h->t), P.lo_vid_d, P.lo_lane_d, h->stream);
        h->n_launch += 1;
        CK(h, cudaMemcpyAsync(ov.data(), P.lo_vid_d, ov.size() * 4, cudaMemcpyDeviceToHost, h->stream));
        CK(h, cudaMemcpyAsync(ol.data(), P.lo_lane_d, ol.size(), cudaMemcpyDeviceToHost, h->stream));
        CK(h, cudaStreamSynchronize(h->stream));
        std::vector<int> cnt(nt), icnt(nt);
        CK(h, cudaMemcpy(cnt.data(), P.cnt[par], nt * 4, cudaMemcpyDeviceToHost));
        CK(h, cudaMemcpy(icnt.data(), P.icnt[par], nt * 4, cudaMemcpyDeviceToHost));
        for (int T : P.tiles)
          for (int i = 0; i < cnt[T] + icnt[T]; ++i) {
            const size_t p = (size_t)h->tile_base[T] + i;
            per[h->tile_lanes[h->tile_lane_off[T] + ol[p]]].push_back(ov[p]);
          }
      }
    } else {
      // global view across processes: the (s, vid) order of the gathered state
      for (int k = 0; k < nv; ++k) if (status[k] == ST_DRIVING) per[lane[k]].push_back(k);
      for (int l = 0; l < h->nl; ++l)
        std::sort(per[l].begin(), per[l].end(), [&](int a, int b) {
          return vs[a] != vs[b] ? vs[a] < vs[b] : a < b;
        });
    }
    int off = 0;
    for (int l = 0; l < h->nl; ++l) {
      o->lane_offsets[l] = off;
      for (int k : per[l]) o->lane_order[off++] = k;
    }
    o->lane_offsets[h->nl] = off;
  }
  return SIM_OK;
}

sim_status sim_read_state(sim_handle h, sim_state *o) { return read_state_impl(h, o, false); }

sim_status sim_read_state_device(sim_handle h, sim_state *o) {
  sim_status st = check(h);
  if (st) return st;
  if (!o || !o->status || !o->lane || !o->cursor || !o->wait_steps || !o->insert_time ||
      !o->arrive_time || !o->s || !o->v)
    return fail(h, SIM_E_INVALID, "sim_read_state_device needs the vid-indexed device buffers");
  if (h->ipc) return fail(h, SIM_E_INVALID, "sim_read_state_device: one process (use sim_read_state_global across processes)");
  std::vector<StepArgs> parts;
  for (Part &P : h->parts) parts.push_back(step_args(P, h->t));
  launch_state_device(parts.data(), (int)parts.size(), h->nv, o->status, o->lane, o->cursor,
                      o->wait_steps, o->insert_time, o->arrive_time, o->s, o->v, h->stream);
  h->n_launch += 1 + 2 * (int64_t)parts.size();
  Part &P0 = h->parts[0];
  const size_t nj = h->nj;
  if (nj) {
    if (o->junc_policy) CK(h, cudaMemcpyAsync(o->junc_policy, P0.SG.policy, nj, cudaMemcpyDeviceToDevice, h->stream));
    if (o->junc_phase) CK(h, cudaMemcpyAsync(o->junc_phase, P0.SG.phase, nj * 4, cudaMemcpyDeviceToDevice, h->stream));
    if (o->junc_elapsed) CK(h, cudaMemcpyAsync(o->junc_elapsed, P0.SG.elapsed, nj * 4, cudaMemcpyDeviceToDevice, h->stream));
    if (o->junc_yellow_left) CK(h, cudaMemcpyAsync(o->junc_yellow_left, P0.SG.yellow_left, nj * 4, cudaMemcpyDeviceToDevice, h->stream));
    if (o->junc_pending) CK(h, cudaMemcpyAsync(o->junc_pending, P0.SG.pending, nj * 4, cudaMemcpyDeviceToDevice, h->stream));
    if (o->junc_remaining) CK(h, cudaMemcpyAsync(o->junc_remaining, P0.SG.remaining, nj * 4, cudaMemcpyDeviceToDevice, h->stream));
  }
  if (o->lane_signal) CK(h, cudaMemcpyAsync(o->lane_signal, P0.A.lane_sig, h->nl, cudaMemcpyDeviceToDevice, h->stream));
  if (o->lane_dir) {
    st = push_staging(h, h->dir.data(), h->nl, o->lane_dir);
    if (st) return st;
  }
  o->t = h->t;
  return SIM_OK;
}
sim_status sim_read_state_global(sim_handle h, sim_state *o) { return read_state_impl(h, o, true); }

sim_status sim_read_decisions(sim_handle h, sim_decisions *o) {
  sim_status st = check(h);
  if (st) return st;
  if (!h->P.record_decisions) return fail(h, SIM_E_INVALID, "created without record_decisions");
  st = device_check(h);
  if (st) return st;
  const size_t n = h->nv;
  std::vector<int32_t> lead(n), of(n), side(4 * n);
  std::vector<int8_t> hops(n), ph(n), lc(n), hand(n), fin(n), ins(n);
  std::vector<float> acc(n);
  std::vector<uint8_t> guard(n), mark(n);
  std::vector<int32_t> t32(4 * n);
  std::vector<int8_t> t8(n);
  std::vector<float> tf(n);
  std::vector<uint8_t> tu(n), tm(n);
  for (Part &P : h->parts) {
    const StepArgs &A = P.A;
    CK(h, cudaMemcpy(tm.data(), A.r_mark, n, cudaMemcpyDeviceToHost));
    auto take32 = [&](const int32_t *src, std::vector<int32_t> &dst, size_t w) -> sim_status {
      CK(h, cudaMemcpy(t32.data(), src, w * n * 4, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < n; ++k) if (tm[k]) for (size_t q = 0; q < w; ++q) dst[w * k + q] = t32[w * k + q];
      return SIM_OK;
    };
    auto take8 = [&](const int8_t *src, std::vector<int8_t> &dst) -> sim_status {
      CK(h, cudaMemcpy(t8.data(), src, n, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < n; ++k) if (tm[k]) dst[k] = t8[k];
      return SIM_OK;
    };
    take32(A.r_leader, lead, 1); take32(A.r_of, of, 1); take32(A.r_side, side, 4);
    take8(A.r_hops, hops); take8(A.r_phantom, ph); take8(A.r_lc, lc); take8(A.r_hand, hand);
    take8(A.r_fin, fin);
    CK(h, cudaMemcpy(t8.data(), A.r_ins, n, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < n; ++k) ins[k] |= t8[k];
    CK(h, cudaMemcpy(tf.data(), A.r_acc, n * 4, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < n; ++k) if (tm[k]) acc[k] = tf[k];
    CK(h, cudaMemcpy(tu.data(), A.r_guard, n, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < n; ++k) if (tm[k]) guard[k] = tu[k];
  }
  if (o->leader_vid) std::memcpy(o->leader_vid, lead.data(), n * 4);
  if (o->leader_hops) std::memcpy(o->leader_hops, hops.data(), n);
  if (o->phantom) std::memcpy(o->phantom, ph.data(), n);
  if (o->old_follower_vid) std::memcpy(o->old_follower_vid, of.data(), n * 4);
  if (o->side_vid) std::memcpy(o->side_vid, side.data(), 4 * n * 4);
  if (o->lc) std::memcpy(o->lc, lc.data(), n);
  if (o->handoffs) std::memcpy(o->handoffs, hand.data(), n);
  if (o->accel) std::memcpy(o->accel, acc.data(), n * 4);
  if (o->finished) std::memcpy(o->finished, fin.data(), n);
  if (o->inserted) std::memcpy(o->inserted, ins.data(), n);
  if (o->guard) std::memcpy(o->guard, guard.data(), n);
  return SIM_OK;
}

sim_status sim_read_metrics(sim_handle h, sim_metrics *m) {
  sim_status st = check(h);
  if (st) return st;
  if (!m) return fail(h, SIM_E_INVALID, "out is NULL");
  // everything is enqueued first and read back through one pinned buffer, so
  // a read costs one synchronisation of the stream
  const bool lanes = m->lane_count || m->lane_waiting_at_end || m->road_avg_speed;
  const size_t ncnt = (size_t)(kNAcc + 3) * h->parts.size();
  const size_t bytes = ncnt * 8 + (lanes ? (2 * (size_t)h->nl + h->nr) * 4 : 0);
  if (h->rd_cap < bytes) {
    CK(h, cudaStreamSynchronize(h->stream));
    if (h->rd_pinned) cudaFreeHost(h->rd_pinned);
    h->rd_pinned = nullptr;
    CK(h, cudaHostAlloc(&h->rd_pinned, bytes, cudaHostAllocDefault));
    h->rd_cap = bytes;
  }
  long long *hc = reinterpret_cast<long long *>(h->rd_pinned);
  int32_t *hl = reinterpret_cast<int32_t *>(hc + ncnt);
  for (Part &P : h->parts) {
    StepArgs a = step_args(P, h->t);
    launch_reduce_acc(P.A.tacc, h->nt, a.cnt_in, a.icnt_in, P.A.status, 0, P.red_d, h->stream);
    h->n_launch += 1;
  }
  if (h->comm || h->ipc) {
    sim_status st = allreduce_sum(h, 0, 0, 0, kNAcc + 3);
    if (st) return st;
  }
  for (size_t q = 0; q < h->parts.size(); ++q)
    CK(h, cudaMemcpyAsync(hc + q * (kNAcc + 3), h->parts[q].red_d, (kNAcc + 3) * 8,
                          cudaMemcpyDeviceToHost, h->stream));
  bool lane_direct[3] = {false, false, false};
  if (lanes) {
    Part &P0 = h->parts[0];
    int32_t *d = P0.lanestat_d;
    // every lane belongs to one tile: the loopback partitions together write all
    // of them; ranks of a real partition only their own, so zero first
    float *rs = m->road_avg_speed ? reinterpret_cast<float *>(d + 2 * (size_t)h->nl) : nullptr;
    if (h->comm || h->ipc) CK(h, cudaMemsetAsync(d, 0, (2 * (size_t)h->nl + h->nr) * 4, h->stream));
    for (Part &P : h->parts) {
      StepArgs a = step_args(P, h->t);
      launch_lane_stats(a, d, d + h->nl, rs, h->P.queue_zone_m, h->stream);
      h->n_launch += 1;
    }
    if (h->comm || h->ipc) {
      st = allreduce_sum(h, 1, 1, 0, 2 * (int64_t)h->nl);
      if (!st && rs) st = allreduce_sum(h, 1, 2, 2 * (int64_t)h->nl, h->nr);
      if (st) return st;
    }
    // each lane array straight into the caller's buffer when that is pinned
    // host memory (no staging copy), else through the pinned staging buffer
    void *dst[3] = {m->lane_count, m->lane_waiting_at_end, m->road_avg_speed};
    const size_t off[3] = {0, (size_t)h->nl, 2 * (size_t)h->nl};
    const size_t cnt[3] = {(size_t)h->nl, (size_t)h->nl, (size_t)h->nr};
    for (int q = 0; q < 3; ++q) {
      if (!dst[q]) continue;
      cudaPointerAttributes pa{};
      const bool pinned = cudaPointerGetAttributes(&pa, dst[q]) == cudaSuccess && pa.type == cudaMemoryTypeHost;
      if (!pinned) cudaGetLastError();            // clear a possible "invalid value" from the query
      CK(h, cudaMemcpyAsync(pinned ? dst[q] : (void *)(hl + off[q]), d + off[q], cnt[q] * 4,
                            cudaMemcpyDeviceToHost, h->stream));
      lane_direct[q] = pinned;                    // done: no staging copy below
    }
  }
  st = device_check(h);
  if (st) return st;
  std::vector<long long> c(kNAcc + 3, 0);
  for (size_t q = 0; q < h->parts.size(); ++q)
    for (int k = 0; k < kNAcc + 3; ++k) c[k] += hc[q * (kNAcc + 3) + k];
  if (c[ACC_OVERFLOW] > 0) {
    h->sticky = SIM_E_CAPACITY;
    return fail(h, SIM_E_CAPACITY, "a road-tile inbox or a migration buffer overflowed its capacity");
  }
  m->t = h->t;
  m->n_driving = c[kNAcc];
  m->n_finished = h->fin0 + (c[ACC_FINISHED] - h->acc_fin0);
  m->n_pending = h->nv - m->n_driving - m->n_finished;
  m->vehicle_steps = c[ACC_VEH_STEPS];
  m->sum_travel_steps = c[ACC_SUM_TRAVEL];
  m->sum_wait_steps_finished = c[ACC_SUM_WAIT_FIN];
  m->sum_depart_delay = c[ACC_SUM_DELAY];
  m->n_lane_changes = c[ACC_LANE_CHANGES];
  m->n_handoffs = c[ACC_HANDOFFS];
  m->n_inserted = c[ACC_INSERTED];
  m->n_guard_hits = c[ACC_GUARD];
  m->att_finished = c[ACC_FINISHED] ? (double)c[ACC_SUM_TRAVEL] / (double)c[ACC_FINISHED] : 0.0;
  // ATT over all vehicles (ledger L27): the sum of insert_time over the
  // DRIVING vehicles is the loaded sum plus ACC_SUM_INSERT since (+insert_time
  // at every insertion, -insert_time at every arrival)
  m->sum_time_driving = (int64_t)h->t * m->n_driving - (h->ins0 + (c[ACC_SUM_INSERT] - h->acc_ins0));
  {
    const long long n_all = c[ACC_FINISHED] + m->n_driving;
    m->att_all = n_all ? (double)(c[ACC_SUM_TRAVEL] + m->sum_time_driving) / (double)n_all : 0.0;
  }
  if (m->lane_count && !lane_direct[0]) std::memcpy(m->lane_count, hl, h->nl * 4);
  if (m->lane_waiting_at_end && !lane_direct[1]) std::memcpy(m->lane_waiting_at_end, hl + h->nl, h->nl * 4);
  if (m->road_avg_speed && !lane_direct[2]) std::memcpy(m->road_avg_speed, hl + 2 * (size_t)h->nl, h->nr * 4);
  return SIM_OK;
}

sim_status sim_read_group_metrics(sim_handle h, int32_t n_groups, sim_metrics *out) {
  sim_status st = check(h);
  if (st) return st;
  if (!out) return fail(h, SIM_E_INVALID, "out is NULL");
  if (!h->n_groups || n_groups != h->n_groups)
    return fail(h, SIM_E_INVALID, "the handle has no road_group or a different n_groups");
  std::vector<long long> c;
  st = read_group_counters(h, c);
  if (st) return st;
  for (int g = 0; g < h->n_groups; ++g) {
    const long long *x = c.data() + (size_t)g * (kNAcc + 1);
    sim_metrics &m = out[g];
    m.t = h->t;
    m.n_driving = x[kNAcc];
    m.n_finished = h->grp_fin0[g] + (x[ACC_FINISHED] - h->grp_acc_fin0[g]);
    m.n_pending = h->grp_nv[g] - m.n_driving - m.n_finished;
    m.vehicle_steps = x[ACC_VEH_STEPS];
    m.sum_travel_steps = x[ACC_SUM_TRAVEL];
    m.sum_wait_steps_finished = x[ACC_SUM_WAIT_FIN];
    m.sum_depart_delay = x[ACC_SUM_DELAY];
    m.n_lane_changes = x[ACC_LANE_CHANGES];
    m.n_handoffs = x[ACC_HANDOFFS];
    m.n_inserted = x[ACC_INSERTED];
    m.n_guard_hits = x[ACC_GUARD];
    m.att_finished = x[ACC_FINISHED] ? (double)x[ACC_SUM_TRAVEL] / (double)x[ACC_FINISHED] : 0.0;
    m.sum_time_driving = 0;                         // per-group trips in progress: not reduced
    m.att_all = 0.0;
  }
  return SIM_OK;
}

sim_status sim_enable_timing(sim_handle h, int32_t enable) {
  sim_status st = check(h);
  if (st) return st;
  st = device_check(h);
  if (st) return st;
  h->timing = enable != 0;
  h->ev_used = 0;
  h->n_launch = 0;
  return SIM_OK;
}

sim_status sim_read_timing(sim_handle h, double *step_ms, double *signal_ms, int64_t *n_launches) {
  sim_status st = check(h);
  if (st) return st;
  st = device_check(h);
  if (st) return st;
  double ks = 0, sg = 0;
  for (size_t i = 0; i + 3 <= h->ev_used; i += 3) {
    float a = 0, b = 0;
    CK(h, cudaEventElapsedTime(&a, h->ev_pool[i], h->ev_pool[i + 1]));
    CK(h, cudaEventElapsedTime(&b, h->ev_pool[i + 1], h->ev_pool[i + 2]));
    sg += a;
    ks += b;
  }
  if (step_ms) *step_ms = ks;
  if (signal_ms) *signal_ms = sg;
  if (n_launches) *n_launches = h->n_launch;
  return SIM_OK;
}

sim_status sim_load_state(sim_handle h, const sim_state *in) {
  return sim_load_state_inbox(h, in, nullptr);
}

sim_status sim_load_state_inbox(sim_handle h, const sim_state *in, const uint8_t *to_inbox) {
  sim_status st = check(h);
  if (st) return st;
  if (!in || !in->status || !in->lane || !in->cursor || !in->wait_steps || !in->insert_time ||
      !in->arrive_time || !in->s || !in->v || !in->lane_dir ||
      (h->nj && (!in->junc_policy || !in->junc_phase || !in->junc_elapsed ||
                 !in->junc_yellow_left || !in->junc_pending)))
    return fail(h, SIM_E_INVALID, "sim_load_state needs every state field");
  st = device_check(h);
  if (st) return st;
  HostState S;
  const int nv = h->nv;
  S.t = in->t;
  S.status.assign(in->status, in->status + nv);
  S.lane.assign(in->lane, in->lane + nv);
  S.cursor.assign(in->cursor, in->cursor + nv);
  S.wait.assign(in->wait_steps, in->wait_steps + nv);
  S.insert_time.assign(in->insert_time, in->insert_time + nv);
  S.arrive_time.assign(in->arrive_time, in->arrive_time + nv);
  S.s.assign(in->s, in->s + nv);
  S.v.assign(in->v, in->v + nv);
  for (int k = 0; k < nv; ++k) {
    if (S.status[k] > 2) return fail(h, SIM_E_RANGE, "bad status");
    if (S.status[k] != ST_DRIVING) continue;
    int l = S.lane[k];
    if (l < 0 || l >= h->nl) return fail(h, SIM_E_RANGE, "lane out of range");
    int c = S.cursor[k];
    if (c < 0 || c >= h->rlen[k]) return fail(h, SIM_E_RANGE, "cursor out of range");
    if (!(S.s[k] >= 0 && S.s[k] <= h->L[l]) || !(S.v[k] >= 0))
      return fail(h, SIM_E_RANGE, "s/v out of range for vehicle " + std::to_string(k));
  }
  for (int j = 0; j < h->nj; ++j)
    if (in->junc_policy[j] > POL_MAXP) return fail(h, SIM_E_RANGE, "junction policy out of range");
  S.jpol.assign(in->junc_policy, in->junc_policy + h->nj);
  S.jphase.assign(in->junc_phase, in->junc_phase + h->nj);
  S.jel.assign(in->junc_elapsed, in->junc_elapsed + h->nj);
  S.jy.assign(in->junc_yellow_left, in->junc_yellow_left + h->nj);
  S.jpend.assign(in->junc_pending, in->junc_pending + h->nj);
  if (in->junc_remaining) S.jrem.assign(in->junc_remaining, in->junc_remaining + h->nj);
  else S.jrem.assign(h->nj, -1);
  S.dir.assign(in->lane_dir, in->lane_dir + h->nl);
  if (to_inbox) S.to_inbox.assign(to_inbox, to_inbox + nv);
  return upload_state(h, S);
}

sim_status sim_partition(const sim_graph *g, const sim_trips *tr, const sim_params *p,
                         int32_t *road_owner, int32_t *plan_sizes) {
  // Host-only: the partition and exchange plan sim_create would use (no GPU needed).
  sim_s *h = new sim_s();
  sim_status st = validate_and_copy(h, g, tr, p);
  if (!st) st = build_tiles(h);
  if (!st) {
    h->world = std::max(1, p->world);
    if (p->road_owner) h->tile_owner.assign(p->road_owner, p->road_owner + h->nr);
    else h->tile_owner = h->world > 1 ? default_partition(h, h->world) : std::vector<int>(h->nr, 0);
    if (road_owner) std::memcpy(road_owner, h->tile_owner.data(), h->nr * 4);
    if (plan_sizes && h->world > 1) {
      Plan plan = make_plan(h);
      const int W = h->world;
      for (int a = 0; a < W; ++a)
        for (int b = 0; b < W; ++b) {
          plan_sizes[2 * (a * W + b)] = plan.mig_cap[a][b];
          plan_sizes[2 * (a * W + b) + 1] = (int32_t)plan.halo[a][b].size();
        }
    }
  } else {
    g_create_err = h->err;
  }
  delete h;
  return st;
}

sim_status sim_destroy(sim_handle h) {
  {
    std::lock_guard<std::mutex> lk(g_live_mu);
    if (!h || !g_live.erase(h)) return SIM_E_STATE;     // destroyed twice / never created
  }
  destroy_impl(h);
  return SIM_OK;
}

const char *sim_last_error(sim_handle h) {
  return (h && is_live(h)) ? h->err.c_str() : g_create_err.c_str();
}

}  // extern "C"
