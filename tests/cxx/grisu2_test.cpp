// grisu2_test.cpp -- include/wgpf_grisu2.h against the reference's JSON
// library (nlohmann/json 3.11.3, the dependency export_chrome_trace prints
// its doubles with): byte-identical number text for random doubles of every
// exponent and for trace-like values cycles / cycles_per_us.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "json.hpp"
#include "wgpf_grisu2.h"

int main(int argc, char** argv) {
  const long iters = argc > 1 ? atol(argv[1]) : 1000000;
  std::mt19937_64 rng(argc > 2 ? atol(argv[2]) : 7);
  long n = 0, bad = 0;
  auto check = [&](double x) {
    const std::string a = nlohmann::json(x).dump();
    char b[64];
    const int l = wgpf_json::format_double(b, x);
    ++n;
    if (a != std::string(b, l)) {
      if (bad < 5) printf("mismatch %.17g json=%s ours=%.*s\n", x, a.c_str(), l, b);
      ++bad;
    }
  };
  for (long t = 0; t < iters; ++t) {
    const uint64_t cyc = rng() >> (rng() % 64);
    const double cpu = t % 3 == 0 ? 1000.0 : (t % 3 == 1 ? 1965.0 : 1.0 + (rng() % 100000) / 7.0);
    check((double)cyc / cpu);
    const uint64_t bits = rng();
    double y;
    memcpy(&y, &bits, 8);
    if (std::isfinite(y)) check(y);
  }
  for (double z : {0.0, -0.0, 1.0, 0.1, 1e15, 1e16, 123456789012345.0, 5e-324,
                   1.7976931348623157e308, 1e-5, 0.0001, 2.2250738585072014e-308})
    check(z);
  printf("n=%ld bad=%ld\n", n, bad);
  return bad != 0;
}
