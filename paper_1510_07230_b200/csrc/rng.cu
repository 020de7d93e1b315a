// Host restatement of the reference's portable generator (rng.hpp:13-41):
// std::mt19937_64, 53-bit bits->double, Box-Muller with a spare. Produces the
// reference's exact bits, so the GPU path starts from the very same u0 as the
// CPU reference for a given seed (tests/problems.hpp:59-68). Also a device fill
// (counter-based, not the reference's bits) for measurement blocks (C5).
#include <algorithm>
#include <cmath>
#include <random>

#include "kernels.h"

namespace po {

void rng_normals_slab(uint64_t seed, int N, int64_t ng_full, int64_t offset, int64_t count,
                      double* out) {
  // The stream is one sequence of Box-Muller pairs over the flat orbital-major
  // index k = i * ng_full + p (the spare of a pair crosses orbital rows). A rank
  // keeps points [offset, offset + count) of every orbital; pairs with neither
  // value in its slab only advance the engine (the u1 == 0 redraw included) —
  // std::mt19937_64 cannot skip ahead cheaply, but the transcendentals can be.
  std::mt19937_64 eng(seed);
  auto uniform = [&]() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
  auto keep = [&](int64_t k) {
    const int64_t p = k % ng_full;
    return p >= offset && p < offset + count;
  };
  const int64_t total = (int64_t)N * ng_full;
  for (int64_t k = 0; k < total; k += 2) {
    double u1 = uniform();
    while (u1 == 0.0) u1 = uniform();
    const double u2 = uniform();
    const bool k0 = keep(k), k1 = k + 1 < total && keep(k + 1);
    if (!k0 && !k1) continue;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.141592653589793 * u2;
    if (k0) out[(k / ng_full) * count + (k % ng_full - offset)] = r * std::cos(theta);
    if (k1) out[((k + 1) / ng_full) * count + ((k + 1) % ng_full - offset)] = r * std::sin(theta);
  }
}

// initialize_orbitals' draws (optimizer.cpp:156-197) for one attempt seed:
// per orbital a width uniform(0.5, 2.0), then one uniform(-1, 1) per grid point
// scaled by 1e-2, in the reference's order. Keeps the slab [offset, offset+count).
void rng_init_noise_slab(uint64_t seed, int N, int64_t ng_full, int64_t offset, int64_t count,
                         double* widths, double* noise) {
  std::mt19937_64 eng(seed);
  auto uniform = [&]() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
  for (int i = 0; i < N; ++i) {
    widths[i] = 0.5 + (2.0 - 0.5) * uniform();
    double* o = noise + (int64_t)i * count;
    for (int64_t p = 0; p < ng_full; ++p) {
      const double v = 1e-2 * (-1.0 + (1.0 - -1.0) * uniform());
      if (p >= offset && p < offset + count) o[p - offset] = v;
    }
  }
}

namespace {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// i.i.d. N(0,1) from a counter hash of (seed, global point index, orbital):
// Box-Muller on two 53-bit uniforms; independent of the slab decomposition
__global__ void fill_normal_kernel(double* __restrict__ out, int N, int64_t ngl, int64_t ld,
                                   int64_t gofs, int64_t ng_full, uint64_t seed) {
  const int i = blockIdx.y;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < ngl;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = (uint64_t)i * (uint64_t)ng_full + (uint64_t)(gofs + p);
    const uint64_t a = mix64(seed ^ (key * 0x9E3779B97F4A7C15ull));
    const uint64_t b = mix64(a ^ 0xD1B54A32D192ED03ull);
    const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = (double)(b >> 11) * 0x1.0p-53;
    out[(int64_t)i * ld + p] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  }
}
}  // namespace

void launch_fill_normal(const SlabGeom& g, int N, int64_t ng_full, uint64_t seed, double* out,
                        cudaStream_t s) {
  dim3 grid((unsigned)std::min<int64_t>((g.ngl + 255) / 256, 4096), (unsigned)N);
  ::po::count_launch();
  fill_normal_kernel<<<grid, 256, 0, s>>>(out, N, g.ngl, g.ld, g.z0 * g.plane, ng_full, seed);
}

}  // namespace po
