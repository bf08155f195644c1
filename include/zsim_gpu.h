/*
 * zsim_gpu.h -- C-ABI of the B200-native batched driving-simulator step.
 *
 * This is the drop-in boundary for the reference's `zsim::sim::Env`
 * (/root/reference/proj/src/core/simcore.hpp:191-245).  The reference builds a
 * hidden-visibility C-API shared library `zsim` from capi/zsim_capi.cpp
 * (proj/src/CMakeLists.txt:24-27) whose sources are not shipped, so the entry
 * points below are designed fresh: plain pointers and sizes, no C++ or torch
 * types, CUDA streams passed as `void*` (a `cudaStream_t`).  Every entry point
 * cites the reference interface it replaces.
 *
 * Layouts:
 *   - state   : SoA over the batch (SimStateBatch, simcore.hpp:107-121); the
 *               reference's AoS EgoState (dynamics.hpp:10-16) is split into
 *               x/y/heading/v/steering arrays.
 *   - stepout : SoA (StepOut, simcore.hpp:123-131); `event` is DoneReason u8.
 *   - obs     : row-major [B][slot][feat] f32 per modality, byte-identical to
 *               ObservationBatch (simcore.hpp:76-103).
 *   - actions : int32 [B] accel / steer bin indices (Env::step,
 *               simcore.hpp:215-216).
 *
 * Errors: every function returns a status.  Codes 1..4 follow the order of
 * zsim::ErrorKind (common.hpp:13); 5 is a CUDA failure.  zsim_last_error()
 * returns a thread-local message for the last failing call on this thread.
 */
#ifndef ZSIM_GPU_H_
#define ZSIM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define ZSIM_API __attribute__((visibility("default")))
#else
#define ZSIM_API
#endif

#define ZSIM_ABI_VERSION 2

enum zsim_status {
    ZSIM_OK = 0,
    ZSIM_INVALID_ARGUMENT = 1, /* ErrorKind::invalid_argument */
    ZSIM_CONFIG = 2,           /* ErrorKind::config */
    ZSIM_IO = 3,               /* ErrorKind::io */
    ZSIM_RUNTIME = 4,          /* ErrorKind::runtime */
    ZSIM_CUDA = 5
};

/* DoneReason (simcore.hpp:47-54). */
enum zsim_done_reason {
    ZSIM_REASON_NONE = 0,
    ZSIM_REASON_COLLISION = 1,
    ZSIM_REASON_OFF_ROUTE = 2,
    ZSIM_REASON_RED_LIGHT = 3,
    ZSIM_REASON_STOP_LINE = 4,
    ZSIM_REASON_GOAL_REACHED = 5
};

/* SimConfig (simcore.hpp:14-45) + dyn::Limits (dynamics.hpp:18-21). */
typedef struct zsim_sim_config {
    double wheelbase;
    double ego_length;
    double ego_width;
    double ego_center_offset;
    double delta_max;
    double v_min;
    double goal_radius;
    double footprint_margin;
    double stop_cross_speed;
    double stop_zone;
    double stop_slow_speed;
    int32_t disable_dones;
    int32_t n_agents;
    int32_t n_road;
    int32_t n_route;
    double w_progress;
    double w_speed;
    double w_lat;
    double w_lon;
    double terminal_penalty;
    double feature_radius;
    int32_t threads; /* accepted for API parity; the device ignores it */
    int32_t reserved;
} zsim_sim_config;

/* SimStateBatch (simcore.hpp:107-121), SoA.  The same struct describes host
 * buffers and device buffers; `stopped_flags` has env->total_stop_lines
 * entries, every other array has `batch` entries. */
typedef struct zsim_state_view {
    double* x;
    double* y;
    double* heading;
    double* v;
    double* steering;
    int32_t* t;
    uint8_t* done;
    uint8_t* reason;
    uint64_t* rng;
    double* proj_s;
    double* proj_d;
    uint8_t* proj_in_corridor;
    uint8_t* events;
    uint8_t* stopped_flags;
} zsim_state_view;

/* StepOut (simcore.hpp:123-131). */
typedef struct zsim_stepout_view {
    float* reward;
    uint8_t* event;
    float* s;
    float* a_lat;
    float* a_lon;
    float* v;
} zsim_stepout_view;

/* ObservationBatch (simcore.hpp:76-103): active [B][9], agents [B][n_agents][6],
 * road [B][n_road][12], route [B][n_route][5], value_only [B][2]. */
typedef struct zsim_obs_view {
    float* active;
    float* agents;
    float* road;
    float* route;
    float* value_only;
} zsim_obs_view;

/* Shape summary of an environment (Env accessors, simcore.hpp:200-209). */
typedef struct zsim_env_info {
    int32_t batch;            /* B = ScenarioBatch::batch */
    int32_t horizon;          /* ScenarioBatch::horizon (padded T) */
    double dt;                /* ScenarioBatch::dt */
    int32_t total_stop_lines; /* length of stopped_flags */
    int32_t zero_accel_idx;   /* ActionTable::nearest_accel(0) */
    int32_t zero_steer_idx;   /* ActionTable::nearest_steer(0) */
    int32_t num_accel;
    int32_t num_steer;
    /* per-batch padded capacities of the device pack */
    int32_t cap_steps, cap_agents, cap_road, cap_route, cap_lanes, cap_vertices, cap_lights, cap_stops;
    int32_t device;
    uint64_t static_bytes; /* device bytes of the immutable scenario pack */
    int32_t scenarios;     /* scenarios staged (== batch unless controlled) */
    int32_t controlled;    /* 1: rows are controlled actors (zsim_env_create_controlled) */
    int32_t step_observe_kernels; /* kernels one zsim_step_observe launches (launch policy) */
    int32_t reserved0;
} zsim_env_info;

typedef struct zsim_env zsim_env;

ZSIM_API int zsim_abi_version(void);
ZSIM_API const char* zsim_last_error(void);

/* SimConfig{} defaults (simcore.hpp:14-45). */
ZSIM_API int zsim_sim_config_defaults(zsim_sim_config* cfg);

/* Env::Env(shared_ptr<const ScenarioBatch>, SimConfig, ActionTable)
 * (simcore.hpp:193-194, simcore.cpp:203-233), with the batch given the way the
 * reference builds it: load_batch(Dataset(path), indices, horizon)
 * (scenario_io.cpp:439-445) over an in-memory ZSIM container image
 * (scenario.hpp:97-104, scenario_io.cpp:319-394).  `indices` may be NULL to
 * take every record in order.  Bins NULL => ActionTable::defaults()
 * (dynamics.cpp:21-26).  Route frames, stop/light s, goal_s, initial_s,
 * logged_progress and route border points are staged on the host in fp64 with
 * the reference's operation order, then uploaded once. */
ZSIM_API int zsim_env_create(const uint8_t* zsim_file, size_t nbytes, const int64_t* indices, int32_t n_indices,
                             int32_t horizon, const zsim_sim_config* cfg, const double* accel_bins, int32_t n_accel,
                             const double* steer_bins, int32_t n_steer, int32_t device, zsim_env** out);
/* "All agents controlled" (the reference has no such
 * mode, its ego-only path is simcore.cpp:300-304).  Same arguments as
 * zsim_env_create; the env has one row per controllable actor of every
 * scenario (actor 0 = the logged ego, actor k = agent k-1; an agent is
 * controllable when valid at every logged step), scenario-major.  Row
 * (s, j) is exactly a reference Env row over the scenario that
 * zsim_controlled_expand writes for it: ego log = actor j's log, goal 4 m past
 * its last logged point along its last heading, every other actor
 * log-replayed in actor order (the logged ego as an agent with the SimConfig
 * ego box).  Roadgraph, route corridor, lights and stop lines are staged once
 * per scenario and shared by its rows. */
ZSIM_API int zsim_env_create_controlled(const uint8_t* zsim_file, size_t nbytes, const int64_t* indices,
                                        int32_t n_indices, int32_t horizon, const zsim_sim_config* cfg,
                                        const double* accel_bins, int32_t n_accel, const double* steer_bins,
                                        int32_t n_steer, int32_t device, zsim_env** out);
/* Row table: scenario index (into the staged scenarios) and controlled actor
 * (-1 in ego mode) of each of the env's `batch` rows; either may be NULL. */
ZSIM_API int zsim_env_get_rows(const zsim_env* env, int32_t* scenario, int32_t* actor);
/* The per-row scenarios of zsim_env_create_controlled as a ZSIM container
 * image (row order), for running the reference Env on exactly those rows.
 * Free with zsim_free_buffer. */
ZSIM_API int zsim_controlled_expand(const uint8_t* zsim_file, size_t nbytes, const int64_t* indices,
                                    int32_t n_indices, const zsim_sim_config* cfg, uint8_t** out_buf,
                                    size_t* out_len);
ZSIM_API int zsim_env_destroy(zsim_env* env);

/* BatchStream (scenario_stream.hpp:12-40): the dataset
 * in file order as batches of `batch_size` (the last may be short), each
 * staged as a device Env.  With `prefetch`, batch k+1 is decoded, staged on
 * the host and uploaded from pinned memory on a copy stream while the caller
 * simulates batch k; delivered batches are identical either way.
 * `controlled` = stage each batch like zsim_env_create_controlled. */
typedef struct zsim_stream zsim_stream;
ZSIM_API int zsim_stream_create(const uint8_t* zsim_file, size_t nbytes, int32_t batch_size, int32_t horizon,
                                const zsim_sim_config* cfg, const double* accel_bins, int32_t n_accel,
                                const double* steer_bins, int32_t n_steer, int32_t device, int32_t prefetch,
                                int32_t controlled, zsim_stream** out);
ZSIM_API int zsim_stream_num_batches(const zsim_stream* stream, int64_t* out);
/* The next batch's Env, owned by the stream and valid until the next call (or
 * destroy); *env = NULL once the dataset is exhausted. */
ZSIM_API int zsim_stream_next(zsim_stream* stream, zsim_env** env);
ZSIM_API int zsim_stream_destroy(zsim_stream* stream);
ZSIM_API int zsim_env_get_info(const zsim_env* env, zsim_env_info* out);
/* Env::goal_s / initial_s / logged_progress (simcore.hpp:207-209): host arrays of B doubles (any may be NULL). */
ZSIM_API int zsim_env_get_scalars(const zsim_env* env, double* goal_s, double* initial_s, double* logged_progress);

/* Device buffers (caller-owned; one contiguous allocation per call). */
ZSIM_API int zsim_state_alloc(zsim_env* env, zsim_state_view* dev_out);
ZSIM_API int zsim_state_free(zsim_env* env, zsim_state_view* dev);
ZSIM_API int zsim_stepout_alloc(zsim_env* env, zsim_stepout_view* dev_out);
ZSIM_API int zsim_stepout_free(zsim_env* env, zsim_stepout_view* dev);
ZSIM_API int zsim_obs_alloc(zsim_env* env, zsim_obs_view* dev_out);
ZSIM_API int zsim_obs_free(zsim_env* env, zsim_obs_view* dev);

/* Blob layouts: every view the library allocates is carved from one
 * contiguous block.  Carving caller memory (e.g. pinned host memory from
 * zsim_host_alloc) with the same layout lets a copy between the two move as a
 * single DMA. */
ZSIM_API int zsim_layout_bytes(const zsim_env* env, size_t* state_bytes, size_t* stepout_bytes, size_t* obs_bytes);
ZSIM_API int zsim_state_carve(const zsim_env* env, void* base, zsim_state_view* out);
ZSIM_API int zsim_stepout_carve(const zsim_env* env, void* base, zsim_stepout_view* out);
ZSIM_API int zsim_obs_carve(const zsim_env* env, void* base, zsim_obs_view* out);
/* Page-locked host memory (cudaHostAlloc) for the host-vector path. */
ZSIM_API int zsim_host_alloc(size_t bytes, void** out);
ZSIM_API int zsim_host_free(void* p);

/* Copies between views; `dir` 0 = host->device, 1 = device->host,
 * 2 = device->device.  Asynchronous on `stream` (host buffers should be pinned
 * for overlap). */
ZSIM_API int zsim_state_copy(zsim_env* env, const zsim_state_view* dst, const zsim_state_view* src, int32_t dir,
                             void* stream);
ZSIM_API int zsim_stepout_copy(zsim_env* env, const zsim_stepout_view* dst, const zsim_stepout_view* src,
                               int32_t dir, void* stream);
ZSIM_API int zsim_obs_copy(zsim_env* env, const zsim_obs_view* dst, const zsim_obs_view* src, int32_t dir,
                           void* stream);

/* ---- device fast path (all pointers device pointers, stream-ordered) ---- */

/* Env::init_state(seed) (simcore.cpp:237-276). */
ZSIM_API int zsim_reset(zsim_env* env, uint64_t seed, const zsim_state_view* out, void* stream);

/* Env::step(state, accel_idx, steer_idx, next, out) (simcore.cpp:406-421).
 * `out` may alias `in`.  Out-of-range action indices (dynamics.cpp:66-71) set
 * the env's device error word and leave that row unchanged; the error is
 * reported by zsim_check_errors(). */
ZSIM_API int zsim_step(zsim_env* env, const zsim_state_view* in, const int32_t* accel_idx, const int32_t* steer_idx,
                       const zsim_state_view* out, const zsim_stepout_view* so, void* stream);

/* Env::observe(state, obs) (simcore.cpp:540-552). */
ZSIM_API int zsim_observe(zsim_env* env, const zsim_state_view* in, const zsim_obs_view* obs, void* stream);

/* Fused Env::step followed by Env::observe of the stepped state, one kernel
 * (the rollout loop body, simcore.cpp:590-609). */
ZSIM_API int zsim_step_observe(zsim_env* env, const zsim_state_view* in, const int32_t* accel_idx,
                               const int32_t* steer_idx, const zsim_state_view* out, const zsim_stepout_view* so,
                               const zsim_obs_view* obs, void* stream);

/* Optional device buffer of int32 [B][n_agents + n_road + n_route] that the
 * observe kernels fill with the selected candidate indices (agent index into
 * Scenario::agents, flat road-feature point index in nearest_features order
 * (roads.cpp:220-229), route border point index (simcore.cpp:181-200)); -1 for
 * empty slots.  NULL disables.  Used by the parity suite. */
ZSIM_API int zsim_set_debug_topk(zsim_env* env, int32_t* dev_idx);

/* Kernel arrangement of step+observe / observe: 0 = automatic (one fused
 * kernel, except batches deeper than three waves of rows on the GPU -- eight
 * for controlled-row envs -- which run step+agents and road/route top-k as
 * separate kernels),
 * 1 = always fused, 2 = always split.  Results are identical; only speed
 * differs. */
ZSIM_API int zsim_set_launch_policy(zsim_env* env, int32_t policy);
/* Synchronises `stream`, reads and clears the device error word.  Returns
 * ZSIM_INVALID_ARGUMENT ("action index out of range") if any step since the
 * last check saw a bad action index, else ZSIM_RUNTIME if any step produced a
 * non-finite ego state (NaN / Inf: failure detection, the step itself is
 * unchanged -- the reference does not check). */
ZSIM_API int zsim_check_errors(zsim_env* env, void* stream);

/* Episode-stats vector of a state (the counts behind
 * metrics::Aggregate, metrics.hpp:56-69): int64[8] = {rows, done rows,
 * rows with latched collision, off_route, red_light, stop_line, goal_reached
 * event bits, sum over rows of (proj_s - initial_s) in micrometres}.  Integer
 * so a cross-GPU ncclAllReduce(sum) is exact.  `out_dev` is device memory. */
/* ---- Device rollout recording --------------------
 * EpisodeBatch (simcore.hpp:167-186) in device memory: [B][T] row-major
 * arrays (index b*horizon + t) and B-vectors. */
typedef struct zsim_episode_view {
    int32_t* accel_idx;
    int32_t* steer_idx;
    float* logp;
    float* value;
    float* reward;
    float* s;
    float* a_lat;
    float* a_lon;
    float* v;
    uint8_t* done;
    uint8_t* mask;
    float* bootstrap;       /* [B] */
    uint8_t* terminal;      /* [B] DoneReason */
    uint8_t* events;        /* [B] */
    float* initial_s;       /* [B] */
    float* logged_progress; /* [B] */
    int32_t horizon;        /* T of these buffers */
    int32_t reserved;
} zsim_episode_view;

/* One device allocation for an EpisodeBatch of `horizon` steps. */
ZSIM_API int zsim_episode_alloc(zsim_env* env, int32_t horizon, zsim_episode_view* out);
ZSIM_API int zsim_episode_free(zsim_env* env, zsim_episode_view* ep);
/* Bytes of one EpisodeBatch blob and carving of caller memory (host or device)
 * into a view; copies between carved views are single DMAs (dir 0 h2d, 1 d2h, 2 d2d). */
ZSIM_API int zsim_episode_bytes(const zsim_env* env, int32_t horizon, size_t* bytes);
ZSIM_API int zsim_episode_carve(const zsim_env* env, int32_t horizon, void* base, zsim_episode_view* out);
ZSIM_API int zsim_episode_copy(const zsim_env* env, const zsim_episode_view* dst, const zsim_episode_view* src,
                               int32_t dir, void* stream);
/* Env::rollout(ScriptedPolicy, horizon, seed) (simcore.cpp:554-618 with
 * simcore.cpp:69-84) on the device: `accel` / `steer` are a device action
 * script [script_len][B] (time-major) read at each row's state.t (the zero
 * action past its end, as ScriptedPolicy); logp and value are 0 (the scripted
 * policy's PolicyOut).  Records every EpisodeBatch field into `ep`; `obs`
 * (NULL or horizon+1 device observation views) receives obs[0..T-1] and the
 * final observation; `final_state` (NULL or a device state) receives the
 * final state.  Stream-ordered, graph-capturable; bad action indices are
 * reported by zsim_check_errors. */
ZSIM_API int zsim_rollout(zsim_env* env, uint64_t seed, int32_t horizon, const int32_t* accel, const int32_t* steer,
                          int32_t script_len, const zsim_episode_view* ep, const zsim_obs_view* obs,
                          const zsim_state_view* final_state, void* stream);

/* ---- Episode metrics on the device (metrics.cpp:13-131) ---- */
typedef struct zsim_score_bounds {
    double progress, collision, off_route, stop_line, traffic_light, comfort;
} zsim_score_bounds;
typedef struct zsim_comfort_weights {
    double w_accel, w_jerk;
} zsim_comfort_weights;
ZSIM_API int zsim_score_defaults(zsim_score_bounds* bounds, zsim_comfort_weights* weights);
/* Per-row MetricReport (metrics.hpp:25-38), device [B] arrays; any may be NULL. */
typedef struct zsim_metric_view {
    double* relative_progress_raw;
    double* relative_progress;
    double* collision_free;
    double* off_route_free;
    double* stop_line_free;
    double* traffic_light_free;
    double* mixed_comfort;
    double* scenario_score;
    uint8_t* degenerate;
    uint8_t* failed;
    uint8_t* goal_reached;
} zsim_metric_view;
/* Aggregate partial sums: [non-degenerate rows, degenerate rows, sum score,
 * sum relative_progress, sum raw ratio, sum collision_free, sum off_route_free,
 * sum stop_line_free, sum traffic_light_free, sum comfort, failed rows, goal rows]. */
#define ZSIM_AGG_LEN 12
/* score_episode for every row of `ep` + this GPU's Aggregate partial sums
 * (fixed-order reduction: deterministic for a given B) into device double[12]. */
ZSIM_API int zsim_episode_metrics(zsim_env* env, const zsim_episode_view* ep, const zsim_score_bounds* bounds,
                                  const zsim_comfort_weights* weights, const zsim_metric_view* rows, double* sums_dev,
                                  void* stream);
/* metrics::aggregate (metrics.cpp:97-131) from `n_parts` host partial-sum
 * vectors summed in order (e.g. rank order after an all-gather): out12 =
 * [scenarios, degenerate, mean_score, mean_relative_progress,
 * mean_progress_ratio_raw, mean_collision_free, mean_off_route_free,
 * mean_stop_line_free, mean_traffic_light_free, mean_comfort, failure_rate, goal_rate]. */
ZSIM_API int zsim_aggregate_finalize(const double* sums, int32_t n_parts, double* out12);

#define ZSIM_STATS_LEN 8
ZSIM_API int zsim_episode_stats(zsim_env* env, const zsim_state_view* state, int64_t* out_dev, void* stream);

/* ---- host-vector path (the drop-in overloads; synchronous) ---- */

/* Env::init_state(seed) into host buffers. */
ZSIM_API int zsim_reset_host(zsim_env* env, uint64_t seed, const zsim_state_view* out_host);
/* Env::step with host vectors: validates shapes/indices first (throws
 * invalid_argument like simcore.cpp:409-411 / dynamics.cpp:67-69), copies
 * state and actions in, runs the step kernel, copies next state and StepOut out. */
ZSIM_API int zsim_step_host(zsim_env* env, const zsim_state_view* in_host, const int32_t* accel_idx,
                            const int32_t* steer_idx, const zsim_state_view* out_host,
                            const zsim_stepout_view* so_host);
/* Env::observe with host vectors. */
ZSIM_API int zsim_observe_host(zsim_env* env, const zsim_state_view* in_host, const zsim_obs_view* obs_host);
/* Env::step followed by Env::observe of the next state (the rollout loop
 * body, simcore.cpp:590-609) with host vectors, in one call: the state is
 * uploaded once, step and observation run fused, and the observation of one
 * row chunk streams to the host while the next chunk runs.  Same checks and
 * results as zsim_step_host + zsim_observe_host. */
ZSIM_API int zsim_step_observe_host(zsim_env* env, const zsim_state_view* in_host, const int32_t* accel_idx,
                                    const int32_t* steer_idx, const zsim_state_view* out_host,
                                    const zsim_stepout_view* so_host, const zsim_obs_view* obs_host);


/* train::cut_sequences (train/replay.cpp:8-52) output: every sequence is
 * `seq_len` steps (TransitionSequence, train/replay.hpp:14-26); padded steps
 * are zero with mask 0.  obs has capacity * seq_len rows ([seq][k]); the
 * per-step arrays are [capacity][seq_len]; `row` is the episode row b of the
 * sequence (its scenario), `t0` its first step; `count` (device int32) is the
 * number of sequences written. */
typedef struct zsim_sequences_view {
    int32_t capacity;
    int32_t seq_len;
    zsim_obs_view obs;
    int32_t* accel_idx;
    int32_t* steer_idx;
    float* logmu;
    float* reward;
    uint8_t* done;
    uint8_t* mask;
    float* bootstrap; /* [capacity] */
    int32_t* row;     /* [capacity] */
    int32_t* t0;      /* [capacity] */
    int32_t* count;   /* [1] */
} zsim_sequences_view;

/* Device buffers for up to batch * ceil(horizon / seq_len) sequences. */
ZSIM_API int zsim_sequences_alloc(zsim_env* env, int32_t horizon, int32_t seq_len, zsim_sequences_view* out);
ZSIM_API int zsim_sequences_free(zsim_env* env, zsim_sequences_view* seq);
/* cut_sequences(ep, seq_len) (train/replay.cpp:8-52) on the device: `ep` a
 * recorded device EpisodeBatch, `obs` its horizon observation views
 * (obs[t] precedes step t, as zsim_rollout records them).  Sequences come in
 * the reference's order (row-major, then t0); a row stops at its first
 * masked window start.  ZSIM_INVALID_ARGUMENT for seq_len <= 0 (as the
 * reference) or an undersized output.  Stream-ordered. */
ZSIM_API int zsim_cut_sequences(zsim_env* env, const zsim_episode_view* ep, const zsim_obs_view* obs,
                                int32_t seq_len, const zsim_sequences_view* out, void* stream);

/* ---- on-device policy inference ------------------
 * NNPolicy::act (train/policy.hpp:27-58) over forward_row
 * (nn/model.hpp:464-585): the perceiver-style encoder (self attention over
 * the 17 latent tokens, cross attention to road / route / active tokens),
 * the policy and value trunks and heads, then argmax or sampling per row.
 * Parameters are the reference's flat Model<float>::params in ParamIndex
 * order (nn/model.hpp:101-167; matrices column-major as Eigen maps them). */

/* ModelConfig (nn/model.hpp:20-27) with its ObsSpec. */
typedef struct zsim_model_config {
    int32_t latent;       /* 128 */
    int32_t heads;        /* 2 */
    int32_t trunk_blocks; /* 2 */
    int32_t value_embed;  /* 32 */
    int32_t n_agents;     /* ObsSpec: 16 */
    int32_t n_road;       /* 128 */
    int32_t n_route;      /* 64 */
    int32_t n_accel;      /* 7 */
    int32_t n_steer;      /* 5 */
    int32_t reserved;
} zsim_model_config;

typedef struct zsim_policy zsim_policy;

/* ModelConfig{} defaults. */
ZSIM_API int zsim_model_config_defaults(zsim_model_config* cfg);
/* Model::param_count (nn/model.hpp:181); ZSIM_CONFIG for configurations the
 * device kernels are not built for (ModelConfig::validate, model.hpp:29-36). */
ZSIM_API int zsim_policy_param_count(const zsim_model_config* cfg, int64_t* out);
/* Model::init(seed) (nn/model.hpp:199-212) on the host, bit-exact. */
ZSIM_API int zsim_policy_init_params(const zsim_model_config* cfg, uint64_t seed, float* out, int64_t n);
/* PolicySnapshot -> device weights (train/policy.hpp:12-15, 21-22). */
ZSIM_API int zsim_policy_create(const zsim_model_config* cfg, const float* params, int64_t n, int32_t device,
                                zsim_policy** out);
ZSIM_API int zsim_policy_destroy(zsim_policy* policy);
/* NNPolicy::act on HOST buffers (the RolloutPolicy interface,
 * simcore.hpp:144-149): obs rows [0, batch) and rng [batch] uploaded, the
 * device policy run, accel / steer / logp / value [batch] and the advanced
 * rng streams written back.  Synchronous. */
ZSIM_API int zsim_policy_act_host(zsim_policy* policy, const zsim_obs_view* obs, int32_t batch, uint64_t* rng,
                                  int32_t use_argmax, int32_t* accel, int32_t* steer, float* logp, float* value);
/* Arithmetic of the token-tile projections and trunks: 1 (default) = fp32
 * CUDA cores (the reference's Model<float> arithmetic); 0 = tcgen05 tensor
 * cores, tf32 operands, fp32 accumulation (faster; logits ~1e-4 from fp32, so
 * actions can differ where a decision margin is that small).  Everything else
 * is fp32 in both modes. */
ZSIM_API int zsim_policy_set_precision(zsim_policy* policy, int32_t mode);
/* Env::rollout(NNPolicy, horizon, seed) (simcore.cpp:554-618 with
 * train/policy.hpp:27-58) entirely on the device: per step observe -> policy
 * (argmax or sampling with the rows' rng streams) -> step, recording every
 * EpisodeBatch field (logp / value from the policy) into `ep`; the bootstrap
 * is the policy's value on the final observation.  `obs` / `final_state` as
 * zsim_rollout.  Stream-ordered, graph-capturable after one warm-up call. */
ZSIM_API int zsim_rollout_policy(zsim_env* env, zsim_policy* policy, int32_t use_argmax, uint64_t seed,
                                 int32_t horizon, const zsim_episode_view* ep, const zsim_obs_view* obs,
                                 const zsim_state_view* final_state, void* stream);
/* NNPolicy::act (train/policy.hpp:27-58) on device buffers: obs rows [0, batch)
 * of a device observation view; rng [batch] is the per-row stream
 * (SimStateBatch::rng), advanced in place when sampling (unused for argmax).
 * Outputs accel / steer / logp / value [batch]; logits (nullable)
 * [batch][n_accel + n_steer].  Stream-ordered; the first call at a larger
 * batch than before allocates scratch (synchronising), later calls are
 * graph-capturable. */
ZSIM_API int zsim_policy_act(zsim_policy* policy, const zsim_obs_view* obs, int32_t batch, uint64_t* rng,
                             int32_t use_argmax, int32_t* accel, int32_t* steer, float* logp, float* value,
                             float* logits, void* stream);

/* ---- synthetic stress scenarios ---- */

typedef struct zsim_stress_config {
    int32_t count;          /* scenarios */
    int32_t num_steps;      /* logged states per scenario (92) */
    int32_t agents;         /* A: total agents incl. the ego => A-1 logged agents */
    int32_t road_points;    /* P: total road-feature points */
    int32_t lanes;          /* route lanes (4) */
    int32_t lane_vertices;  /* vertices per lane border (64) */
    double dt;              /* 0.1 */
    double speed_limit;     /* 10 m/s */
    double lane_width;      /* 3.5 m */
    int32_t first_index;    /* global index of the first scenario (shards of one global set) */
    int32_t flags;          /* bit 0: C2 actors -- every agent valid at all steps, same-direction route lanes */
} zsim_stress_config;

ZSIM_API int zsim_stress_config_defaults(zsim_stress_config* cfg);
/* Generates scenarios first_index .. first_index+count-1 of the global set
 * deterministically from `seed` (scenario i draws from the stream
 * Rng(seed).split(i), common.hpp:47-50, in closed form) and returns a
 * ZSIM container image in a malloc'd buffer (free with zsim_free_buffer). */
ZSIM_API int zsim_stress_generate(const zsim_stress_config* cfg, uint64_t seed, uint8_t** out_buf, size_t* out_len);
ZSIM_API void zsim_free_buffer(void* buf);
/* A device Env over stress scenarios [first_index, first_index+count) built
 * without a ZSIM image (the scenes are generated on all host cores and staged
 * directly): the benchmark's C3 / C4 shards.  Identical to zsim_env_create over
 * zsim_stress_generate's image of the same range.  `controlled` as in
 * zsim_env_create_controlled. */
ZSIM_API int zsim_env_create_stress(const zsim_stress_config* stress, uint64_t seed, int32_t horizon,
                                    const zsim_sim_config* cfg, int32_t device, int32_t controlled, zsim_env** out);

/* ---- multi-GPU episode-statistics exchange ----
 * Scenarios are sharded across GPUs with no per-step exchange; once per
 * rollout the int64 stats vector (zsim_episode_stats) is summed over all GPUs
 * with one NCCL all-reduce (exact; the reference AllReducer's fixed-order
 * contract, core/train/transport.hpp:59-61) and the fp64 Aggregate partial
 * sums (zsim_episode_metrics; metrics.hpp:56-69) are all-gathered so each rank
 * adds them in rank order (zsim_aggregate_finalize).  NCCL is dlopen'ed at
 * first use (libnccl.so.2).  Replaces the reference's train::AllReducer
 * (transport.hpp:59-98) for this path. */
#define ZSIM_COMM_ID_BYTES 128
typedef struct zsim_comm zsim_comm;
/* 1 when libnccl.so.2 can be loaded, else 0. */
ZSIM_API int zsim_comm_available(void);
/* One process per GPU: rank 0 makes the id, the caller broadcasts it. */
ZSIM_API int zsim_comm_unique_id(uint8_t id[ZSIM_COMM_ID_BYTES]);
ZSIM_API int zsim_comm_init_rank(const uint8_t id[ZSIM_COMM_ID_BYTES], int32_t nranks, int32_t rank, int32_t device,
                                 zsim_comm** out);
/* One process driving `ndev` GPUs (ncclCommInitAll): out[ndev] communicators;
 * devices NULL = 0..ndev-1.  Use one host thread + stream per GPU (or
 * zsim_comm_group) around the collectives. */
ZSIM_API int zsim_comm_init_all(int32_t ndev, const int32_t* devices, zsim_comm** out);
ZSIM_API int zsim_comm_destroy(zsim_comm* comm);
/* ncclCommGetAsyncError surfaced as a status (ZSIM_RUNTIME on an error). */
ZSIM_API int zsim_comm_check(zsim_comm* comm);
/* In place: stats_dev[n] (int64, device) summed over all ranks, on `stream`. */
ZSIM_API int zsim_stats_allreduce(zsim_comm* comm, int64_t* stats_dev, int32_t n, void* stream);
/* gathered_dev[nranks][n] (fp64, device) = every rank's sums_dev[n], rank order. */
ZSIM_API int zsim_metric_sums_allgather(zsim_comm* comm, const double* sums_dev, int32_t n, double* gathered_dev,
                                        void* stream);
/* ncclGroupStart (begin = 1) / ncclGroupEnd (begin = 0). */
ZSIM_API int zsim_comm_group(int32_t begin);

#ifdef __cplusplus
}
#endif

#endif /* ZSIM_GPU_H_ */
