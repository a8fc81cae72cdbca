// corpus_host.cpp -- host regeneration of the BASELINE synthetic corpora.
//
// TEST / BENCH INFRASTRUCTURE ONLY (like the rest of oracle/): bench.py's
// reference arm builds its input batch with it, so the reference's CPU path
// is timed on exactly the records the GPU arm evaluates, and the GPU tests
// check the device generator against it.  The recipes are the shared header
// paper_2511_00292_b200/csrc/eig33_gen_core.h, which uses only IEEE +,-,*,/,
// sqrt and integer operations; compiled here with -ffp-contract=off (and the
// device side with --fmad=false) the two builds produce identical bits.
#include <stddef.h>
#include <stdint.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "../paper_2511_00292_b200/csrc/eig33_gen_core.h"

extern "C" {

// Records [first, first + n) of config 1..5 with `seed` into out (n x 9
// doubles), on `threads` host threads (contiguous slices).  0 ok, 2 bad argument.
int corpus_generate(int config, uint64_t seed, uint64_t first, size_t n, double* out, int threads) {
  if (config < 1 || config > 5 || (n && !out)) return 2;
  const size_t t = (size_t)std::max(1, std::min(threads, 256));
  auto work = [=](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      const eig33gen::M3 a = eig33gen::make_record(config, seed, first + i);
      for (int k = 0; k < 9; ++k) out[i * 9 + k] = a.e[k];
    }
  };
  if (t == 1 || n < 4096) {
    work(0, n);
    return 0;
  }
  std::vector<std::thread> th;
  for (size_t k = 0; k < t; ++k) th.emplace_back(work, n * k / t, n * (k + 1) / t);
  for (auto& x : th) x.join();
  return 0;
}

}  // extern "C"
