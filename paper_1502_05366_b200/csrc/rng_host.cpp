// rng_host.cpp — the reference's Gaussian stream on the host (parity-mode
// Omega).  Restates reference core/rng.hpp:18-87: splitmix64 seeding
// (:20-24,69-74), xoshiro256++ (:27-38), 53-bit unit doubles (:41),
// Box-Muller with a cached spare (:43-56), substreams (:61-64), column-major
// fill (:82-87).  Built with -ffp-contract=off so the libm pipeline matches
// the reference bit for bit.
#include <cmath>
#include <cstdint>

#include "../../include/rlra_c.h"

namespace {
uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
}  // namespace

extern "C" {

void rlra_rng_seed(rlra_rng* r, uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : r->s) w = splitmix64(x);
    r->spare = 0.0;
    r->have_spare = 0;
}

uint64_t rlra_rng_next_u64(rlra_rng* r) {
    uint64_t* s = r->s;
    const uint64_t out = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
}

double rlra_rng_next_gaussian(rlra_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = 1.0 - static_cast<double>(rlra_rng_next_u64(r) >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(rlra_rng_next_u64(r) >> 11) * 0x1.0p-53;
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    r->spare = radius * std::sin(angle);
    r->have_spare = 1;
    return radius * std::cos(angle);
}

void rlra_rng_substream(rlra_rng* parent, rlra_rng* child) {
    uint64_t key = rlra_rng_next_u64(parent);
    rlra_rng_seed(child, splitmix64(key));
}

void rlra_rng_gaussian_fill(rlra_rng* r, int rows, int cols, double* out) {
    const int64_t n = int64_t(rows) * cols;
    for (int64_t i = 0; i < n; ++i) out[i] = rlra_rng_next_gaussian(r);
}

void rlra_omega_fill_rng(void* user, int, int rows, int cols, double* out) {
    rlra_rng_gaussian_fill(static_cast<rlra_rng*>(user), rows, cols, out);
}

void rlra_omega_fill_rng_substream(void* user, int, int rows, int cols, double* out) {
    rlra_rng child;
    rlra_rng_substream(static_cast<rlra_rng*>(user), &child);
    rlra_rng_gaussian_fill(&child, rows, cols, out);
}

void rlra_omega_fill_rng_nodes(void* user, int draw, int rows, int cols, double* out) {
    rlra_rng_nodes* nd = static_cast<rlra_rng_nodes*>(user);
    const int node = draw >> 16;
    rlra_rng* st = &nd->nodes[node < nd->count ? node : nd->count - 1];
    if (nd->substream_per_draw) {
        rlra_rng child;
        rlra_rng_substream(st, &child);
        rlra_rng_gaussian_fill(&child, rows, cols, out);
    } else {
        rlra_rng_gaussian_fill(st, rows, cols, out);
    }
}

}  // extern "C"
