// TEST INFRASTRUCTURE: the benchmark's synthetic workload for the oracle side.
//
// bench.py's reference arm and cpu_baseline leg must time the reference
// simulator on the same stress scenarios the device arm runs
// without mapping the product library.  This shim compiles the workload
// generator's sources (csrc/zsim_stressgen.cpp, and csrc/zsim_scenario.cpp for
// the ZSIM codec and the C2 per-actor expansion) into
// oracle/_ref/libzsim_stress.so; nothing here is measured.
#include <cstdlib>
#include <cstring>
#include <string>

#include "zsim_gpu.h"
#include "zsim_scenario.hpp"

namespace zs {
std::string stress_generate(const zsim_stress_config& cfg, uint64_t seed);
}

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const zs::Error& e) {
        g_err = e.what();
        return int(e.kind);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

int hand_out(const std::string& img, uint8_t** out, size_t* n) {
    *out = static_cast<uint8_t*>(std::malloc(img.size() ? img.size() : 1));
    if (!*out) return 4;
    std::memcpy(*out, img.data(), img.size());
    *n = img.size();
    return 0;
}
}  // namespace

extern "C" {

const char* zstress_last_error(void) { return g_err.c_str(); }

int zstress_generate(const zsim_stress_config* cfg, uint64_t seed, uint8_t** out, size_t* n) {
    std::string img;
    int rc = guarded([&] { img = zs::stress_generate(*cfg, seed); });
    return rc ? rc : hand_out(img, out, n);
}

// C2: the per-row scenarios of every controllable actor,
// in row order (zsim_controlled_expand of the product, same definition).
int zstress_controlled_expand(const uint8_t* file, size_t nbytes, double ego_length, double ego_width,
                              double ego_center_offset, uint8_t** out, size_t* n) {
    std::string img;
    int rc = guarded([&] {
        zs::ZsimIndex idx = zs::zsim_index(file, nbytes);
        const zs::EgoBoxDims ebd{ego_length, ego_width, ego_center_offset};
        img = zs::zsim_header(idx.dt);
        for (int64_t r = 0; r < int64_t(idx.records.size()); ++r) {
            zs::Scene sc = zs::zsim_decode(file, nbytes, idx, r);
            for (int j = 0; j < zs::num_actors(sc); ++j)
                if (zs::actor_controllable(sc, j)) zs::zsim_encode_append(img, zs::controlled_scene(sc, j, ebd));
        }
    });
    return rc ? rc : hand_out(img, out, n);
}

void zstress_free(void* p) { std::free(p); }
}
