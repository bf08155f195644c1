/*
 * zsim_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference simulator's hot path (reset, step,
 * observe over a batch of ZSIM scenarios) used as the parity checker of the
 * sm_100a kernels.  Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/src/core/).  Built with
 * -ffp-contract=off so its fp64 arithmetic rounds like the reference built the
 * same way; it is pinned against oracle/_ref (the reference compiled in place)
 * and against the committed golden fixtures in tests/golden/.
 *
 * Differences from the reference, by design:
 *   - road points are ordered by (d2, flat index) instead of libstdc++'s
 *     unspecified partial_sort order inside exact d2 ties (roads.cpp:231-232);
 *   - errors are returned as codes (1 invalid_argument, 2 config, 3 io,
 *     4 runtime) with a message, never thrown.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
 */
#ifndef ZSIM_ORACLE_H_
#define ZSIM_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/zsim_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct zor_env zor_env;

const char* zor_last_error(void);
int zor_env_create(const uint8_t* zsim_file, size_t nbytes, const int64_t* indices, int32_t n_indices, int32_t horizon,
                   const zsim_sim_config* cfg, zor_env** out);
void zor_env_destroy(zor_env* env);
int zor_env_info(const zor_env* env, int32_t* batch, int32_t* horizon, int32_t* total_stop_lines);
int zor_scalars(const zor_env* env, double* goal_s, double* initial_s, double* logged_progress);
int zor_init_state(const zor_env* env, uint64_t seed, const zsim_state_view* out);
int zor_step(const zor_env* env, const zsim_state_view* in, const int32_t* accel, const int32_t* steer,
             const zsim_state_view* out, const zsim_stepout_view* so);
/* `topk` (nullable) receives int32 [B][n_agents + n_road + n_route] selected indices, -1 for empty slots. */
int zor_observe(const zor_env* env, const zsim_state_view* in, const zsim_obs_view* obs, int32_t* topk);

#ifdef __cplusplus
}
#endif

#endif
