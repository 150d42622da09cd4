// config4_inputs.cpp — BASELINE config 4's synthetic inputs as a C++ caller generates them
// (std::mt19937_64 seeded 0x5eed5eed, std::uniform_real_distribution<double>; SURVEY §8d draw
// order: per rank u_a, v_a, p_a, then one U(0.9, 1.1) factor per size). Prints the raw draws as
// hex words so tests/test_configs_rng.py can compare them bit for bit with configs.py.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

static void put(double x) {
  std::uint64_t b;
  std::memcpy(&b, &x, 8);
  std::printf("%016llx\n", (unsigned long long)b);
}

int main(int argc, char** argv) {
  const int r = argc > 1 ? std::atoi(argv[1]) : 16;
  const long m = argc > 2 ? std::atol(argv[2]) : 4096;
  std::mt19937_64 rng(0x5eed5eed);
  std::uniform_real_distribution<double> uv(0.5, 1.5), up(-0.5, 0.5), un(0.9, 1.1);
  for (int a = 0; a < r; ++a) {
    put(uv(rng));
    put(uv(rng));
    put(up(rng));
  }
  for (long s = 0; s < m; ++s) put(un(rng));
  return 0;
}
