// Host restatement of the reference's portable generator (rng.hpp:13-41):
// std::mt19937_64, 53-bit bits->double, Box-Muller with a spare. Produces the
// reference's exact bits, so the GPU path starts from the very same u0 as the
// CPU reference for a given seed (tests/problems.hpp:59-68).
#include <cmath>
#include <random>

#include "kernels.h"

namespace po {

void rng_normals_slab(uint64_t seed, int N, int64_t ng_full, int64_t offset, int64_t count,
                      double* out) {
  std::mt19937_64 eng(seed);
  auto uniform = [&]() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
  bool have = false;
  double spare = 0.0;
  auto normal = [&]() {
    if (have) {
      have = false;
      return spare;
    }
    double u1 = uniform();
    while (u1 == 0.0) u1 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.141592653589793 * uniform();
    spare = r * std::sin(theta);
    have = true;
    return r * std::cos(theta);
  };
  for (int i = 0; i < N; ++i) {
    double* o = out + (int64_t)i * count;
    for (int64_t p = 0; p < ng_full; ++p) {
      const double v = normal();
      if (p >= offset && p < offset + count) o[p - offset] = v;
    }
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

}  // namespace po
