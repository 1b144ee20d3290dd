/* oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, serial fp64 CPU simulator of the model in DESIGN.md §1
 * (arXiv 2406.10661, App. A2.2-A2.3; §3.1-3.3).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_2406_10661_b200/csrc/), and the CUDA
 * path never loads it.
 *
 * All structs here are the oracle's own; they intentionally do not reuse
 * include/sim.h.
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n_lanes, n_roads, n_junctions;
  const float *lane_length, *lane_max_speed;
  const int32_t *lane_road, *lane_junction, *lane_left, *lane_right;
  const int32_t *succ_offsets, *succ_lanes;
  const uint8_t *lane_turn, *lane_kind;
  const int32_t *tidal_partner;
  const uint8_t *lane_dir0;
  const int32_t *road_lane_offsets, *road_lanes;
  const int32_t *junc_lane_offsets, *junc_lanes;
  const int32_t *junc_phase_offsets;
  const uint8_t *phase_green;
  const int32_t *phase_green_steps;
  const uint8_t *junc_policy;   /* 0 NONE 1 FIXED_TIME 2 MANUAL 3 MAX_PRESSURE */
  const int32_t *junc_offset_steps;
} or_graph;

typedef struct {
  int32_t n_trips;
  const int32_t *depart_step;
  const uint8_t *on_network_at_t0;
  const int32_t *route_offsets, *route_roads;
  const int32_t *start_lane;
  const float *start_s, *start_v, *end_s;
  const uint8_t *profile;
} or_trips;

typedef struct {
  uint64_t seed;
  int32_t n_profiles;
  const float *profiles;        /* [n_profiles][6] a_max a_comf T s0 v_max len */
  float politeness, b_hard, b_safe, v_wait, queue_zone_m;
  int32_t yellow_steps, lookahead_lanes;
  int32_t store_fp32;           /* round s, v to fp32 after every step */
  int32_t reverse_order;        /* process vehicles in reverse vid order (P-PERM) */
  int32_t max_pressure_period;  /* MAX_PRESSURE decision period in steps (<= 0: 30) */
} or_params;

typedef struct {
  int32_t t;
  /* vid-indexed [n_trips] */
  uint8_t *status;              /* 0 PENDING 1 DRIVING 2 FINISHED */
  int32_t *lane, *cursor, *wait_steps, *insert_time, *arrive_time;
  double *s, *v;
  /* junction-indexed */
  uint8_t *junc_policy;
  int32_t *junc_phase, *junc_elapsed, *junc_yellow_left, *junc_pending;
  int32_t *junc_remaining;      /* MANUAL set_tl_duration steps left, -1 none */
  /* lane-indexed */
  uint8_t *lane_dir;
  uint8_t *lane_signal;         /* signals seen by vehicles in the last step */
} or_state;

typedef struct {                /* decisions of the last step, vid-indexed */
  int32_t *leader_vid;          /* -1 none */
  int8_t *leader_hops;          /* 0 in-lane, h lanes ahead, -1 none */
  int8_t *phantom;              /* 1 stop-line phantom active (current lane) */
  int32_t *old_follower_vid;
  int32_t *side_vid;            /* [4*n]: LF LB RF RB of the current lane */
  int8_t *lc;                   /* -1 left, 0 stay, +1 right */
  int8_t *handoffs;
  double *accel;                /* acceleration used */
  int8_t *finished;             /* 1 arrived this step */
  int8_t *inserted;             /* 1 inserted this step */
} or_decisions;

typedef struct {
  int32_t t;
  int64_t n_pending, n_driving, n_finished;
  int64_t vehicle_steps, sum_travel_steps, sum_wait_steps_finished;
  int64_t sum_depart_delay, n_lane_changes, n_handoffs, n_inserted;
  int64_t sum_time_driving;          /* sum over DRIVING vehicles of (t - insert_time) */
} or_metrics;

/* returns NULL on invalid input, with a message in err */
void *or_create(const or_graph *g, const or_trips *tr, const or_params *p,
                char *err, int32_t errlen);
void or_destroy(void *h);
int32_t or_step(void *h, int32_t n);
void or_read_state(void *h, or_state *out);
void or_load_state(void *h, const or_state *in);
/* per-lane (s, vid) order of DRIVING vehicles: offsets [n_lanes+1], vids */
void or_lane_order(void *h, int32_t *offsets, int32_t *vids);
void or_read_decisions(void *h, or_decisions *out);
void or_read_metrics(void *h, or_metrics *out);
/* lane_count, lane_waiting_at_end [n_lanes] */
void or_lane_stats(void *h, int32_t *lane_count, int32_t *lane_waiting);
int32_t or_set_signal_phase(void *h, int32_t junction, int32_t phase);
int32_t or_set_lane_direction(void *h, int32_t lane, int32_t dir);
int32_t or_set_signal_policy(void *h, int32_t junction, int32_t policy);
int32_t or_set_signal_duration(void *h, int32_t junction, int32_t steps);
int32_t or_set_vehicle_route(void *h, int32_t vid, int32_t n, const int32_t *roads, float end_s);
int32_t or_set_lane_max_speed(void *h, int32_t lane, float v);
int32_t or_set_lane_restriction(void *h, int32_t lane, int32_t flag);
/* [n_roads] mean speed of the vehicles on each road (free-flow if empty) */
void or_road_avg_speed(void *h, double *out);
/* Philox4x32-10 block function, exposed for the known-answer test (P-RNG) */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double or_u53(uint64_t seed, int32_t vid, int32_t t);
/* IDM, exposed for closed-form pins */
double or_idm(double v, double v0, int32_t has_leader, double gap, double dv,
              double a_max, double a_comf, double T, double s0, double b_hard);
double or_p_lc(double u_total);

#ifdef __cplusplus
}
#endif
#endif
