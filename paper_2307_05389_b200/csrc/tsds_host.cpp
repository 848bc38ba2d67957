// tsds_host.cpp -- host-side binning for host-resident x.
//
// When x lives in host memory only the ~27 probes per bin edge of the
// reference's binary search touch it, so the library bins on the host and
// ships nothing but y (and the offsets) over PCIe.  Same semantics as the
// device kernels in tsds_bin.cuh and the reference binning.py:43-82 /
// _kernels.py:506-535 (numba arithmetic typing for the uniform check).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/tsds.h"

namespace {

template <class T, class D>
int uniform_t(const void* xv, int64_t n) {
  const T* x = (const T*)xv;
  if (n < 2) return 0;
  D d = (D)x[1] - (D)x[0];
  if constexpr (std::is_same<T, int64_t>::value) {
    if (!((int64_t)d > 0)) return 0;
  } else {
    if (!(d > (D)0)) return 0;
  }
  for (int64_t i = 1; i < n - 1; i++)
    if ((D)x[i + 1] - (D)x[i] != d) return 0;
  return 1;
}

template <class T>
double f64_at(const void* x, int64_t i) {
  return (double)((const T*)x)[i];
}

typedef double (*getter_t)(const void*, int64_t);

getter_t getter(int dt) {
  switch (dt) {
    case 1: return f64_at<float>;
    case 2: return f64_at<double>;
    case 3: return f64_at<int8_t>;
    case 4: return f64_at<int16_t>;
    case 5: return f64_at<int32_t>;
    case 6: return f64_at<int64_t>;
    case 7: return f64_at<uint8_t>;
    case 8: return f64_at<uint16_t>;
    case 9: return f64_at<uint32_t>;
    case 10: return f64_at<uint64_t>;
    default: return nullptr;
  }
}

}  // namespace

extern "C" int tsds_host_is_uniform_spaced(const void* x, int dt, int64_t n) {
  switch (dt) {
    case 1: return uniform_t<float, float>(x, n);
    case 2: return uniform_t<double, double>(x, n);
    case 3: return uniform_t<int8_t, int64_t>(x, n);
    case 4: return uniform_t<int16_t, int64_t>(x, n);
    case 5: return uniform_t<int32_t, int64_t>(x, n);
    case 6: return uniform_t<int64_t, uint64_t>(x, n);  // int64 wraps
    case 7: return uniform_t<uint8_t, int64_t>(x, n);
    case 8: return uniform_t<uint16_t, int64_t>(x, n);
    case 9: return uniform_t<uint32_t, int64_t>(x, n);
    case 10: return uniform_t<uint64_t, uint64_t>(x, n);
    default: return 0;
  }
}

extern "C" int tsds_host_equal_width_offsets(const void* x, int dt, int64_t n, int64_t nb, int64_t* off) {
  getter_t g = getter(dt);
  if (!g || nb < 1) return TSDS_ERR_ARG;
  if (n == 0) {
    for (int64_t k = 0; k <= nb; k++) off[k] = 0;
    return TSDS_OK;
  }
  const double x0 = g(x, 0);
  const double xn = g(x, n - 1);
  const double span = xn - x0;
  if (!std::isfinite(span)) return TSDS_ERR_SPAN;
  if (span == 0.0) {
    for (int64_t k = 0; k < nb; k++) off[k] = 0;
    off[nb] = n;
    return TSDS_OK;
  }
  if (tsds_host_is_uniform_spaced(x, dt, n)) {
    for (int64_t k = 0; k <= nb; k++) off[k] = (int64_t)((unsigned __int128)k * (uint64_t)n / (uint64_t)nb);
    return TSDS_OK;
  }
  auto work = [&](int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; k++) {
      double prod = (double)k * span;
      double q = prod / (double)nb;
      double e = x0 + q;
      int64_t lo = 0, hi = n;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (g(x, mid) < e) lo = mid + 1; else hi = mid;
      }
      off[k] = lo;
    }
  };
  int64_t edges = nb - 1;
  unsigned hw = std::thread::hardware_concurrency();
  int nt = (int)std::min<int64_t>(hw ? hw : 1, std::max<int64_t>(1, edges / 256));
  if (nt > 32) nt = 32;
  if (nt <= 1) {
    work(1, nb);
  } else {
    std::vector<std::thread> th;
    int64_t ch = (edges + nt - 1) / nt;
    for (int t = 0; t < nt; t++) {
      int64_t k0 = 1 + t * ch, k1 = std::min<int64_t>(nb, k0 + ch);
      if (k0 < k1) th.emplace_back(work, k0, k1);
    }
    for (auto& t : th) t.join();
  }
  off[0] = 0;
  off[nb] = n;
  return TSDS_OK;
}
