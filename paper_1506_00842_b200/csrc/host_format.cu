// host_format.cu — the `mltune predict` CSV rows (reference cli.py:346-351:
// f"{index},{format(pred, '.17g')}\n" per configuration, one Python call per
// row) formatted natively on host threads. C's "%.17g" and Python's '.17g'
// both print the correctly rounded 17-significant-digit form, so the bytes are
// identical (tests/test_formats.py checks against a reference-written file).
#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "mltune_b200.h"

extern "C" {

MLT_API int mlt_format_predictions(const int64_t* idx, const double* pred, int64_t n, char* out, int64_t cap,
                                   int64_t* used, int32_t threads) {
  if (n < 0 || !used || (n > 0 && (!idx || !pred || !out))) return MLT_EINVAL;
  *used = 0;
  if (n == 0) return MLT_OK;
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if ((int64_t)nt > (n + 4095) / 4096) nt = (int)((n + 4095) / 4096);
  std::vector<std::string> parts(nt);
  auto work = [&](int t) {
    const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
    std::string& s = parts[t];
    s.reserve((size_t)(hi - lo) * 28);
    char line[64];
    for (int64_t q = lo; q < hi; ++q) {
      const int len = snprintf(line, sizeof line, "%" PRId64 ",%.17g\n", idx[q], pred[q]);
      s.append(line, (size_t)len);
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  int64_t total = 0;
  for (const auto& s : parts) total += (int64_t)s.size();
  if (total > cap) return MLT_EINVAL;
  char* at = out;
  for (const auto& s : parts) {
    std::memcpy(at, s.data(), s.size());
    at += s.size();
  }
  *used = total;
  return MLT_OK;
}

}  // extern "C"
