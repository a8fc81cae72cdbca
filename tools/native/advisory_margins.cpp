// Histogram of x/T = -disc / disc_tolerance over the pending (disc < 0) records of a
// BASELINE config (2^20 records, seed 100+config), the product math compiled for the CPU.
// Build: g++ -O2 -ffp-contract=off -std=c++17 tools/native/advisory_margins.cpp -o /tmp/adv \
//          -Loracle -lcorpus -Wl,-rpath,$PWD/oracle   ;  run: /tmp/adv 4
#include <stddef.h>
#include <stdint.h>
#include <cstdio>
#include <cmath>
#include <vector>
#define EIG33_TABLE_DECL static const
#include "../../paper_2511_00292_b200/csrc/eig33_tables.h"
#include "../../paper_2511_00292_b200/csrc/eig33_math.cuh"
using namespace eig33b;
extern "C" int corpus_generate(int config, uint64_t seed, uint64_t first, size_t n, double* out, int threads);
int main(int argc, char** argv) {
  int cfg = atoi(argv[1]); size_t n = 1u << 20;
  std::vector<double> a(n * 9);
  corpus_generate(cfg, 100 + cfg, 0, n, a.data(), 8);
  long pend = 0, flag = 0; long hist[40] = {0};
  long up_settle = 0;
  for (size_t i = 0; i < n; ++i) {
    const double* m = &a[9 * i];
    Inv v = invariants(m);
    if (!(v.disc < 0)) continue;
    pend++;
    double T = disc_tolerance(m, v.j2, v.j3);
    bool f = v.disc < -T;
    flag += f;
    double r = std::log10(-v.disc / T);
    int b = (int)std::floor(r) + 20; if (b < 0) b = 0; if (b > 39) b = 39;
    hist[b]++;
  }
  printf("cfg %d n %zu pending %ld (%.3f) flag-true %ld (%.3f of pending)\n", cfg, n, pend, pend / (double)n, flag, flag / (double)pend);
  for (int b = 0; b < 40; ++b) if (hist[b]) printf("  log10(x/T) in [%d,%d): %ld\n", b - 20, b - 19, hist[b]);
}
