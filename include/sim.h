/* sim.h — C ABI of the B200-native vehicle-update hot path (arXiv 2406.10661).
 *
 * One simulation timestep of the paper's GPU microscopic traffic simulator
 * (App. A2.2 "Execution Process"): per-lane ordering
 * (P:130), leader / follower / side-neighbour lookup including the
 * successor-lane substitution, IDM car following
 * (P:156-167), randomized MOBIL lane changing, signal response
 * (P:200), integration with hand-off into successor lanes,
 * departure insertion, per-junction signal update (P:140-141,
 * P:836-841) and travel / wait accounting.
 * The exact model (incl. every reading of a silent passage) is DESIGN.md §1.
 *
 * Conventions (all entry points):
 *   - every call returns sim_status; 0 = SIM_OK; nothing throws or aborts;
 *   - input pointers are HOST pointers read during the call and copied; the
 *     library never retains them; all device memory is owned by the library;
 *   - sim_read_* write into CALLER-owned buffers (host memory unless stated);
 *   - sim_step is asynchronous on the handle's stream; device faults and
 *     capacity overflows surface at the next synchronising call
 *     (sim_read_state / sim_read_metrics / sim_sync) and make the handle sticky
 *     (SIM_E_STATE afterwards);
 *   - setters take effect at the next step boundary (stream-ordered);
 *     _batch variants equal the single calls applied in order;
 *   - one controlling host thread per handle; every call makes the handle's
 *     device (params.device) current on the calling thread.
 */
#ifndef SIM_H
#define SIM_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SIM_OK = 0,
  SIM_E_INVALID = 1,   /* input violates a rule of DESIGN.md §1.1 (message via sim_last_error) */
  SIM_E_RANGE = 2,     /* id / index out of range; nothing changed */
  SIM_E_OOM = 3,       /* device allocation failed */
  SIM_E_CUDA = 4,      /* CUDA runtime error (handle becomes sticky) */
  SIM_E_NCCL = 5,      /* reserved: multi-GPU exchange failure */
  SIM_E_STATE = 6,     /* destroyed / sticky handle */
  SIM_E_CAPACITY = 7   /* a per-tile slot or inbox capacity overflowed (sticky) */
} sim_status;

typedef struct sim_s *sim_handle;   /* opaque, owned by the library */

/* Lane graph (App. A2.1).  Host memory, caller-owned, CSR layout.
 * Lanes are road lanes (lane_road >= 0, lane_junction == -1) or junction
 * lanes (lane_road == -1, lane_junction >= 0).  A junction lane has exactly one
 * predecessor and one successor, both road lanes.  Road lanes of a road have
 * equal length and are listed leftmost first in road_lanes. */
typedef struct {
  int32_t n_lanes, n_roads, n_junctions;
  const float *lane_length;          /* [n_lanes] metres, > 0 */
  const float *lane_max_speed;       /* [n_lanes] m/s, > 0 */
  const int32_t *lane_road;          /* [n_lanes] road id or -1 */
  const int32_t *lane_junction;      /* [n_lanes] junction id or -1 */
  const int32_t *lane_left, *lane_right; /* [n_lanes] neighbour lane or -1 (road lanes only) */
  const int32_t *succ_offsets;       /* [n_lanes+1] CSR lane -> successor lanes */
  const int32_t *succ_lanes;
  const uint8_t *lane_turn;          /* [n_lanes] junction lanes: 0 STRAIGHT 1 LEFT 2 RIGHT */
  const uint8_t *lane_kind;          /* [n_lanes] 0 NORMAL 1 DYNAMIC 2 TIDAL */
  const int32_t *tidal_partner;      /* [n_lanes] partner lane of a TIDAL lane or -1 */
  const uint8_t *lane_dir0;          /* [n_lanes] initial direction (DYNAMIC: 0 STRAIGHT 1 LEFT;
                                        TIDAL: 0 FORWARD = usable, 1 BACKWARD) */
  const int32_t *road_lane_offsets;  /* [n_roads+1] */
  const int32_t *road_lanes;         /* leftmost first */
  const int32_t *junc_lane_offsets;  /* [n_junctions+1] */
  const int32_t *junc_lanes;         /* junction lane "slots" */
  const int32_t *junc_phase_offsets; /* [n_junctions+1] CSR junction -> phases */
  const uint8_t *phase_green;        /* for junction j, phase k: row of n_slots(j) bytes,
                                        rows laid out junction by junction, phase by phase */
  const int32_t *phase_green_steps;  /* [n_phases] FIXED_TIME green duration (steps) */
  const uint8_t *junc_policy;        /* [n_junctions] 0 NONE 1 FIXED_TIME 2 MANUAL
                                        3 MAX_PRESSURE */
  const int32_t *junc_offset_steps;  /* [n_junctions] FIXED_TIME cycle offset */
} sim_graph;

/* Trips (P:826 origin, destination, departure, route).  Host, caller-owned. */
typedef struct {
  int32_t n_trips;                   /* vehicle id = trip index */
  const int32_t *depart_step;        /* [n] >= 0 */
  const uint8_t *on_network_at_t0;   /* [n] 1: DRIVING at t = 0 at (start_lane, start_s, start_v) */
  const int32_t *route_offsets;      /* [n+1] CSR trip -> roads */
  const int32_t *route_roads;
  const int32_t *start_lane;         /* [n] lane of route[0] */
  const float *start_s, *start_v, *end_s; /* [n] metres, m/s, metres on the destination road */
  const uint8_t *profile;            /* [n] index into params.profiles */
} sim_trips;

typedef struct { float a_max, a_comf, T, s0, v_max, length; } sim_profile;

typedef struct {
  uint64_t seed;                     /* Philox key (ledger L16) */
  float dt;                          /* must be 1.0 */
  int32_t n_profiles;                /* <= 256 */
  const sim_profile *profiles;
  float politeness, b_hard, b_safe, v_wait, queue_zone_m; /* 0.1, 8, 4, 0.1, 100 */
  int32_t yellow_steps, lookahead_lanes;                  /* 3, 2 */
  int32_t exact_mode;                /* 1: all per-vehicle math in fp64 (test mode) */
  int32_t record_decisions;          /* 1: keep the last step's decisions for sim_read_decisions */
  int32_t device;                    /* CUDA device ordinal */
  void *stream;                      /* cudaStream_t to run on (NULL = library-created stream) */
  /* Spatial partition over `world` partitions.  world <= 1: one
   * partition.  world > 1: either loopback = 1 (all partitions in this handle
   * on `device`, exchanging by device copies; used to test partition
   * invariance) or one process per GPU with the same nccl_id (from
   * sim_get_nccl_unique_id on one rank) and rank in [0, world).  road_owner
   * (optional, [n_roads]) fixes the partition of each road (with its outgoing
   * junction lanes); NULL = the library's breadth-first partitioner.
   * direct = 1: the step kernel stores each
   * mover crossing the cut straight into the owning partition's inbox and
   * folds it into that partition's lane summary, and reads other partitions'
   * summaries in place — no migration / halo exchange step.  With loopback = 1
   * the partitions share this process; with loopback = 0 it is one process per
   * GPU (rank in [0, world), world <= 32, nccl_id unused) whose buffers are
   * mapped by CUDA IPC (NVLink peer memory): every rank calls sim_ipc_export,
   * the blobs are all-gathered in rank order (e.g. with torch.distributed) and
   * passed to sim_ipc_connect before the first step or read; each step then
   * ends with a device barrier over the ranks. */
  int32_t rank, world, loopback, direct;
  const uint8_t *nccl_id;            /* 128 bytes, NCCL mode only */
  const int32_t *road_owner;
  /* MAX_PRESSURE: a green phase is kept for at least
   * this many steps, then the phase of maximum pressure (sum over its green
   * movements of count(predecessor lane) - count(successor lane), DRIVING
   * vehicles in state(t); ties -> lowest index) is chosen, with the yellow
   * steps in between when it changes.  <= 0: 30. */
  int32_t max_pressure_period;
  /* Batched environments (RL workloads P:146):
   * independent networks stepped by one call are passed as one graph with
   * disconnected components.  vehicle_seed [n_trips] / vehicle_rng_id
   * [n_trips] (optional, NULL = params.seed / vid) set the Philox key and
   * counter of each vehicle's draw (ledger L16), so every environment draws
   * exactly as its standalone run; road_group [n_roads] (optional, values in
   * [0, n_groups)) labels roads, and the vehicles whose start lane is on them,
   * for sim_read_group_metrics. */
  const uint64_t *vehicle_seed;
  const int32_t *vehicle_rng_id;
  const int32_t *road_group;
  int32_t n_groups;
  /* Direct transport across processes: a device barrier that waits longer
   * than this (a peer stopped stepping) flags a sticky SIM_E_CUDA instead of
   * hanging.  <= 0: 60000 ms. */
  int32_t barrier_timeout_ms;
  /* Optional device allocator for every buffer the handle keeps (SURVEY
   * §8(b): e.g. the PyTorch caching allocator, so that PyTorch provides the
   * device memory, BASELINE.json north_star).  alloc(bytes, ctx) returns
   * device memory on params.device or NULL; free_(ptr, ctx) releases it at
   * sim_destroy.  Both NULL: cudaMalloc / cudaFree. */
  void *(*alloc)(size_t bytes, void *ctx);
  void (*free_)(void *ptr, void *ctx);
  void *alloc_ctx;
  /* sim_step(n) with n >= 12 replays a CUDA graph of 6 captured steps
   * (launch cost once per 6 steps, programmatic dependent launches between
   * the step kernels); results are identical to stepping one by
   * one.  Nonzero: always launch step by step.  Graphs are never used with
   * the multi-process transports (IPC barrier, NCCL) or while sim_enable_timing
   * is on. */
  int32_t no_step_graphs;
} sim_params;

typedef struct {
  int32_t n_vehicles, n_lanes, n_junctions, n_tiles;
  int64_t device_bytes;              /* device memory held by the handle */
} sim_sizes;

/* Vehicle / junction / lane state, vid-, junction- and lane-indexed.
 * All arrays caller-owned, sized from sim_sizes; any pointer may be NULL to
 * skip that field on read (not on load). */
typedef struct {
  int32_t t;                         /* steps completed */
  uint8_t *status;                   /* 0 PENDING 1 DRIVING 2 FINISHED */
  int32_t *lane, *cursor, *wait_steps, *insert_time, *arrive_time;
  float *s, *v;
  uint8_t *junc_policy;
  int32_t *junc_phase, *junc_elapsed, *junc_yellow_left, *junc_pending;
  int32_t *junc_remaining;           /* MANUAL set_tl_duration green steps left, -1 none
                                        (optional on load: NULL = -1) */
  uint8_t *lane_dir;
  uint8_t *lane_signal;              /* read only: signals seen in the last step */
  int32_t *lane_offsets;             /* read only, optional: [n_lanes+1] per-lane order CSR */
  int32_t *lane_order;               /* read only, optional: [n_vehicles] vids by (s, vid) */
} sim_state;

/* Decisions of the last step (record_decisions = 1), vid-indexed. */
typedef struct {
  int32_t *leader_vid;               /* -1 none */
  int8_t *leader_hops;               /* 0 in-lane, h lanes ahead, -1 none */
  int8_t *phantom;                   /* stop-line phantom active on the current lane */
  int32_t *old_follower_vid;
  int32_t *side_vid;                 /* [4*n] LF LB RF RB */
  int8_t *lc;                        /* -1 left 0 stay +1 right */
  int8_t *handoffs;
  float *accel;
  int8_t *finished, *inserted;
  uint8_t *guard;                    /* 1: decided by the fp64 guard fallback */
} sim_decisions;

typedef struct {
  int32_t t;
  int64_t n_pending, n_driving, n_finished;
  int64_t vehicle_steps;             /* sum over steps of vehicles moved */
  int64_t sum_travel_steps, sum_wait_steps_finished, sum_depart_delay;
  int64_t n_lane_changes, n_handoffs, n_inserted, n_guard_hits;
  double att_finished;               /* sum_travel_steps / n_finished */
  int64_t sum_time_driving;          /* sum over DRIVING vehicles of (t - insert_time) */
  double att_all;                    /* ATT over all vehicles (ledger L27): (sum_travel_steps +
                                        sum_time_driving) / (n_finished + n_driving), trips in
                                        progress counted with their time so far */
  int32_t *lane_count;               /* optional caller buffer [n_lanes] or NULL */
  int32_t *lane_waiting_at_end;      /* optional [n_lanes]: v < v_wait within queue_zone_m */
  float *road_avg_speed;             /* optional [n_roads]: mean speed of the vehicles on the road's
                                        lanes, the road's max lane speed if none */
} sim_metrics;

/* Create a simulation.  Validates the graph and trips
 * (SIM_E_INVALID names the first violated rule), builds road tiles, allocates
 * device memory on params->device and uploads the t = 0 state. */
sim_status sim_create(const sim_graph *g, const sim_trips *trips,
                      const sim_params *params, sim_handle *out);
/* Direct transport across processes (params.direct = 1, loopback = 0).
 * sim_ipc_export writes this rank's CUDA IPC handles (*n_bytes bytes; out =
 * NULL only reports the size) into out[cap].  sim_ipc_connect takes the blobs
 * of all ranks concatenated in rank order (world x n_bytes; this rank's entry
 * is ignored) and maps the peers' buffers; SIM_E_CUDA if a mapping fails.
 * Until it succeeds sim_step and the reads fail with SIM_E_STATE.  A device
 * barrier that waits longer than 60 s (environment SIM_BARRIER_TIMEOUT_MS at
 * create) for a peer makes the handle sticky (SIM_E_STATE at the next
 * synchronising call) instead of hanging. */
sim_status sim_ipc_export(sim_handle h, uint8_t *out, int32_t cap, int32_t *n_bytes);
sim_status sim_ipc_connect(sim_handle h, const uint8_t *blobs, int32_t n_bytes);

/* Dynamic repartitioning (direct = 1 only,
 * SPMD: every rank calls it at the same step with the same argument).
 * road_owner [n_roads] is the new owner of each road tile; NULL = the library
 * rebalances: its breadth-first partition weighted by the vehicles currently
 * on each road tile (+1), summed over the partitions.  At the step boundary
 * each tile that changes owner is handed over on the device (stayers, inbox,
 * lane summaries and counts, pending-queue heads, its vehicles' insert time
 * and status) — results stay bit-identical to an unpartitioned run (P-PART).
 * *moved_tiles (may be NULL) = tiles that changed owner.  Synchronises the
 * stream.  SIM_E_INVALID without the direct transport, SIM_E_RANGE for an
 * owner outside [0, world). */
sim_status sim_repartition(sim_handle h, const int32_t *road_owner, int32_t *moved_tiles);

/* NCCL unique id for a partitioned run (call on one rank, broadcast the 128
 * bytes to all ranks, e.g. with torch.distributed). */
sim_status sim_get_nccl_unique_id(uint8_t out[128]);
/* Host-only (no GPU): the partition sim_create would use for params->world,
 * written to road_owner [n_roads] (may be NULL), and the exchange plan sizes
 * plan_sizes [world*world*2] (may be NULL): for each (a, b) the migrant-buffer
 * capacity a -> b and the number of lanes whose summary a reads from b. */
sim_status sim_partition(const sim_graph *g, const sim_trips *trips, const sim_params *params,
                         int32_t *road_owner, int32_t *plan_sizes);
/* Advance n >= 0 steps (next_step(n)), asynchronously. */
sim_status sim_step(sim_handle h, int32_t n);
/* Block until all enqueued work finished; reports deferred device errors. */
sim_status sim_sync(sim_handle h);
/* MANUAL phase request (set_tl_phase): junction switches to MANUAL,
 * Y yellow steps then `phase`. */
sim_status sim_set_signal_phase(sim_handle h, int32_t junction, int32_t phase);
sim_status sim_set_signal_phase_batch(sim_handle h, int32_t m, const int32_t *junctions,
                                      const int32_t *phases);
/* Lane direction (set_road_lane_plan P:851 / set_lane_restriction P:846):
 * DYNAMIC: 0 STRAIGHT 1 LEFT; TIDAL: 0 FORWARD (usable) 1 BACKWARD, the
 * partner gets the complement.  SIM_E_INVALID for other lanes. */
sim_status sim_set_lane_direction(sim_handle h, int32_t lane, int32_t dir);
sim_status sim_set_lane_direction_batch(sim_handle h, int32_t m, const int32_t *lanes,
                                        const int32_t *dirs);
/* Signal policy (set_tl_policy): 0 NONE 1 FIXED_TIME 2 MANUAL
 * 3 MAX_PRESSURE, applied at the next step before its signals and before
 * phase requests; FIXED_TIME / MAX_PRESSURE restart the current phase's green
 * timer, a running yellow completes.  SIM_E_RANGE for a bad
 * id or policy; a junction without phases stays NONE. */
sim_status sim_set_signal_policy(sim_handle h, int32_t junction, int32_t policy);
sim_status sim_set_signal_policy_batch(sim_handle h, int32_t m, const int32_t *junctions,
                                       const int32_t *policies);
/* Phase duration (set_tl_duration): the junction switches to MANUAL
 * and its current green (the requested phase's, after a yellow) is held for
 * `steps` >= 1 steps from the next step, then it moves to the next phase
 * (with the yellow) and holds it until the next request. */
sim_status sim_set_signal_duration(sim_handle h, int32_t junction, int32_t steps);
sim_status sim_set_signal_duration_batch(sim_handle h, int32_t m, const int32_t *junctions,
                                         const int32_t *steps);
/* Lane max speed (set_lane_max_speed): m/s > 0, from the next step
 * (v0 = min(lane, vehicle), L6).  The lane-start margin keeps its create-time
 * value (L17). */
sim_status sim_set_lane_max_speed(sim_handle h, int32_t lane, float max_speed);
sim_status sim_set_lane_max_speed_batch(sim_handle h, int32_t m, const int32_t *lanes,
                                        const float *max_speeds);
/* Lane restriction (set_lane_restriction): flag 1 = no entry; the lane
 * is not usable (no lane change into it, no junction lane leads into it,
 * DESIGN §1.3); vehicles already on it continue.  flag 0 lifts it. */
sim_status sim_set_lane_restriction(sim_handle h, int32_t lane, int32_t flag);
sim_status sim_set_lane_restriction_batch(sim_handle h, int32_t m, const int32_t *lanes,
                                          const int32_t *flags);
/* Vehicle route (set_vehicle_route): the vehicle's remaining trip
 * becomes roads[0..n) ending at end_s on roads[n-1] (consecutive roads
 * connected).  roads[0] must be the vehicle's current road (a DRIVING vehicle
 * inside a junction also keeps its committed next road as roads[1]; a PENDING
 * vehicle keeps its first road and start lane); the route cursor restarts at
 * 0.  Synchronising (it reads the vehicles' positions); SIM_E_INVALID and no
 * change on any violation (DESIGN L46). */
sim_status sim_set_vehicle_route(sim_handle h, int32_t vid, int32_t n, const int32_t *roads,
                                 float end_s);
sim_status sim_set_vehicle_route_batch(sim_handle h, int32_t m, const int32_t *vids,
                                       const int32_t *route_offsets, const int32_t *roads,
                                       const float *end_s);
/* Sizes of the handle's entities and device memory, for sizing read buffers
 * (no device work). */
sim_status sim_query_sizes(sim_handle h, sim_sizes *out);
/* The simulator's getters (e.g. get_vehicle_speeds; state per vehicle,
 * junction and lane, App. A2.1; the per-lane order of the linked
 * lists, P:803-806 — as the step kernel merges stayers and inbox, a1).
 * Synchronising reads into caller-owned host buffers.  With partitions,
 * sim_read_state reports the vehicles of the partitions in this handle (one
 * process per rank: its own; the others read as PENDING unless they finished
 * here); sim_read_state_global (collective: every rank calls it) reports every
 * partition's vehicles — with the direct transport across processes it reads
 * the peers' buffers through their IPC mappings; otherwise it equals
 * sim_read_state.  Vehicles are vid-indexed, so the result equals a
 * single-partition run's. */
sim_status sim_read_state(sim_handle h, sim_state *out);
/* sim_read_state into DEVICE buffers on params.device (e.g. torch tensors;
 * SURVEY §8(b) on_device): status, lane, cursor, wait_steps, insert_time,
 * arrive_time, s, v (vid-indexed, all required), and optionally the junction
 * arrays, lane_signal and lane_dir.  Asynchronous on the handle's stream (no
 * synchronisation: the values are those of the step boundary at which the
 * call is enqueued); lane_offsets / lane_order are ignored.  One process
 * (world 1 or loopback); SIM_E_INVALID otherwise. */
sim_status sim_read_state_device(sim_handle h, sim_state *out);
sim_status sim_read_state_global(sim_handle h, sim_state *out);
/* The decisions of the last step (record_decisions = 1; test hook of the
 * parity gate): leader / lookahead hops, stop-line phantom
 * (P:200), followers and side neighbours, lane change,
 * hand-offs / arrivals, insertions, acceleration. */
sim_status sim_read_decisions(sim_handle h, sim_decisions *out);
/* Evaluation metrics: counts of pending / driving / finished
 * vehicles, throughput = finished trips, ATT over finished trips
 * and over all vehicles, waiting time, the lane
 * queue lengths and road average speeds on request.
 * With partitions the counters are summed over all of them, so every rank
 * gets the global values.
 * Collective across processes (NCCL or direct transport): every rank must
 * call every read — sim_read_state, _global, _metrics, _group_metrics, and
 * sim_load_state — in the same order with the same optional buffers present
 * (lane statistics / road speeds), since the reductions are collective. */
sim_status sim_read_metrics(sim_handle h, sim_metrics *out);
/* Per-group metrics (params.road_group): out[n_groups], counters of the tiles
 * (roads) of each group and status counts of its vehicles; the lane buffers
 * of out[] are ignored.  SIM_E_INVALID without road_group or on a different
 * n_groups. */
sim_status sim_read_group_metrics(sim_handle h, int32_t n_groups, sim_metrics *out);
/* Replace the whole state (checkpoint / parity hook; the inverse of the
 * getters).  Pending queues are rebuilt from status (ordered by
 * (depart, vid), ledger L25); all fields except lane_signal /
 * lane_offsets / lane_order are required.  SIM_E_CAPACITY if a road tile
 * would hold more vehicles than its record region. */
sim_status sim_load_state(sim_handle h, const sim_state *in);
/* Test hook of sim_load_state: the DRIVING vehicles with to_inbox[vid] = 1 are
 * placed, unsorted, in their tile's inbox (as if they had entered the tile or
 * changed lane in the last step) instead of among its sorted stayers,
 * so a one-step parity test exercises the step kernel's merge (a1)
 * with populated inboxes.  to_inbox: host array [n_vehicles] or NULL (=
 * sim_load_state).  The state itself is the same. */
sim_status sim_load_state_inbox(sim_handle h, const sim_state *in, const uint8_t *to_inbox);
/* Device timing (measurement hook): enable = 1 opens a new window
 * in which every sim_step launch is bracketed by CUDA events on the handle's
 * stream (and resets the launch counter); sim_read_timing (synchronising)
 * returns the summed device time of the step kernels and of the signal
 * kernels in the window, and the number of library kernel launches. */
sim_status sim_enable_timing(sim_handle h, int32_t enable);
sim_status sim_read_timing(sim_handle h, double *step_kernel_ms, double *signal_kernel_ms,
                           int64_t *n_launches);
/* Release every device buffer (through params.free_ when given); every later
 * call on h fails with SIM_E_STATE. */
sim_status sim_destroy(sim_handle h);
/* Last error message of h (NULL h: the calling thread's last create error). */
const char *sim_last_error(sim_handle h);

#ifdef __cplusplus
}
#endif
#endif
