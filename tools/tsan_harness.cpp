// tsan_harness -- the library's host-side concurrency under ThreadSanitizer
// (SURVEY.md §5 "TSAN on the host harness").  Built by tools/tsan.sh against a
// -fsanitize=thread build of libzsim_gpu.so.  Exercises every place the host
// code runs threads: parallel ZSIM decode + staging (zsim_env_create,
// zsim_env_create_stress: parallel_for), the BatchStream prefetch thread
// (zsim_stream_*: batch k+1 staged and uploaded while batch k steps), and
// concurrent Envs on separate host threads (the one-thread-per-GPU layout of
// zsim_multi_gpu, here on one device).  `cpu` mode stops before any CUDA
// call (decode / generation only) so it also runs on a machine without a GPU.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "zsim_gpu.h"

namespace {
void check(int rc, const char* what) {
    if (rc != ZSIM_OK) {
        std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, zsim_last_error());
        std::exit(1);
    }
}

std::vector<uint8_t> stress(int count, int agents, int points, int first) {
    zsim_stress_config sc;
    check(zsim_stress_config_defaults(&sc), "stress defaults");
    sc.count = count;
    sc.agents = agents;
    sc.road_points = points;
    sc.first_index = first;
    uint8_t* p = nullptr;
    size_t n = 0;
    check(zsim_stress_generate(&sc, 7, &p, &n), "stress generate");
    std::vector<uint8_t> v(p, p + n);
    zsim_free_buffer(p);
    return v;
}

// a few fused steps on an env (device buffers from the C-ABI; zero actions)
void run_env(zsim_env* env, int steps) {
    zsim_env_info info;
    check(zsim_env_get_info(env, &info), "info");
    zsim_state_view s0, s1;
    zsim_stepout_view so;
    zsim_obs_view ob;
    check(zsim_state_alloc(env, &s0), "alloc");
    check(zsim_state_alloc(env, &s1), "alloc");
    check(zsim_stepout_alloc(env, &so), "alloc");
    check(zsim_obs_alloc(env, &ob), "alloc");
    // host-vector API for the actions (no cudart in this harness)
    std::vector<int32_t> a(size_t(info.batch), info.zero_accel_idx), s(size_t(info.batch), info.zero_steer_idx);
    size_t sb = 0, sob = 0, obb = 0;
    check(zsim_layout_bytes(env, &sb, &sob, &obb), "layout");
    void *hs0 = nullptr, *hs1 = nullptr, *hso = nullptr;
    check(zsim_host_alloc(sb, &hs0), "host alloc");
    check(zsim_host_alloc(sb, &hs1), "host alloc");
    check(zsim_host_alloc(sob, &hso), "host alloc");
    zsim_state_view h0, h1;
    zsim_stepout_view hso_v;
    check(zsim_state_carve(env, hs0, &h0), "carve");
    check(zsim_state_carve(env, hs1, &h1), "carve");
    check(zsim_stepout_carve(env, hso, &hso_v), "carve");
    check(zsim_reset_host(env, 42, &h0), "reset host");
    for (int t = 0; t < steps; ++t) {
        check(zsim_step_host(env, &h0, a.data(), s.data(), &h1, &hso_v), "step host");
        std::swap(h0, h1);
    }
    // fused host-vector step + observe (copy stream + events)
    {
        void* hob = nullptr;
        check(zsim_host_alloc(obb, &hob), "host alloc");
        zsim_obs_view hob_v;
        check(zsim_obs_carve(env, hob, &hob_v), "carve");
        for (int t = 0; t < steps; ++t) {
            check(zsim_step_observe_host(env, &h0, a.data(), s.data(), &h1, &hso_v, &hob_v), "step_observe host");
            std::swap(h0, h1);
        }
        zsim_host_free(hob);
    }
    check(zsim_reset(env, 42, &s0, nullptr), "reset");
    check(zsim_check_errors(env, nullptr), "errors");
    zsim_host_free(hs0);
    zsim_host_free(hs1);
    zsim_host_free(hso);
    zsim_state_free(env, &s0);
    zsim_state_free(env, &s1);
    zsim_stepout_free(env, &so);
    zsim_obs_free(env, &ob);
}
}  // namespace

int main(int argc, char** argv) {
    const bool cpu = argc > 1 && std::strcmp(argv[1], "cpu") == 0;
    // parallel generation + decode (zsim_controlled_expand decodes on all cores)
    std::vector<uint8_t> img = stress(96, 12, 400, 0);
    {
        uint8_t* p = nullptr;
        size_t n = 0;
        check(zsim_controlled_expand(img.data(), img.size(), nullptr, 0, nullptr, &p, &n), "expand");
        zsim_free_buffer(p);
    }
    if (cpu) {
        std::printf("tsan_harness: cpu paths done\n");
        return 0;
    }
    // parallel staging
    zsim_env* env = nullptr;
    check(zsim_env_create(img.data(), img.size(), nullptr, 0, 0, nullptr, nullptr, 0, nullptr, 0, 0, &env),
          "env create");
    run_env(env, 3);
    zsim_env_destroy(env);
    zsim_stress_config sc;
    check(zsim_stress_config_defaults(&sc), "stress defaults");
    sc.count = 80;
    sc.agents = 10;
    sc.road_points = 300;
    check(zsim_env_create_stress(&sc, 7, 0, nullptr, 0, 0, &env), "env create stress");
    run_env(env, 2);
    zsim_env_destroy(env);
    // BatchStream: prefetch thread staging batch k+1 while batch k steps
    zsim_stream* st = nullptr;
    check(zsim_stream_create(img.data(), img.size(), 20, 0, nullptr, nullptr, 0, nullptr, 0, 0, 1, 0, &st),
          "stream create");
    for (;;) {
        zsim_env* e = nullptr;
        check(zsim_stream_next(st, &e), "stream next");
        if (!e) break;
        run_env(e, 2);
    }
    check(zsim_stream_destroy(st), "stream destroy");
    // concurrent envs on separate host threads (one env per thread)
    std::vector<std::thread> th;
    for (int k = 0; k < 3; ++k)
        th.emplace_back([k] {
            std::vector<uint8_t> im = stress(24, 8, 300, 24 * k);
            zsim_env* e = nullptr;
            check(zsim_env_create(im.data(), im.size(), nullptr, 0, 0, nullptr, nullptr, 0, nullptr, 0, 0, &e),
                  "env create (thread)");
            run_env(e, 3);
            zsim_env_destroy(e);
        });
    for (auto& t : th) t.join();
    std::printf("tsan_harness: all paths done\n");
    return 0;
}
