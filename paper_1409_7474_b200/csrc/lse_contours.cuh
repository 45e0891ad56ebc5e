// Zero-level contours of a dense fp64 field: marching squares on the device,
// segment assembly on the host.
//
// Reference: extract_contours (engine.py:280-294) calls
// skimage.measure.find_contours(phi, 0.0) (scikit-image >= 0.20,
// pkg/pyproject.toml:13; fully_connected='low', positive_orientation='low')
// and maps (row, col) to (col + 0.5, row + 0.5).  find_contours is two steps,
// restated here from scikit-image's published algorithm:
//   1. per 2x2 square, in row-major square order, the case index
//      (ul > 0) + 2 (ur > 0) + 4 (ll > 0) + 8 (lr > 0) selects 0, 1 or 2
//      oriented segments between edge crossings; a crossing on the edge
//      from -> to sits at fraction (0 - from) / (to - from) (0 when the two
//      values are equal); squares with a NaN corner are skipped;
//   2. the segments, in that order, are joined into polylines by exact
//      endpoint equality (dicts of starts / ends); a contour keeps the index
//      of the first segment that created it, and output is in index order.
// Step 1 is embarrassingly parallel and bandwidth-bound (one fp64 read per
// pixel, two counting passes); step 2 is a sequential hash-join over the
// (far fewer) crossing segments and runs on the host.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <deque>
#include <unordered_map>
#include <vector>

namespace lse {

constexpr int kContourThreads = 256;

struct Seg {
  double fr, fc, tr, tc;     // from (row, col) -> to (row, col)
};

__device__ __forceinline__ double ms_fraction(double from, double to) {
  if (to == from) return 0.0;
  return __ddiv_rn(__dsub_rn(0.0, from), __dsub_rn(to, from));
}

// Segments of square (r0, c0); returns how many, degenerate (from == to)
// segments dropped exactly where the assembly would ignore them.
__device__ __forceinline__ int ms_square(double ul, double ur, double ll, double lr, double r0,
                                         double c0, Seg* out) {
  if (isnan(ul) || isnan(ur) || isnan(ll) || isnan(lr)) return 0;
  const int cs = (ul > 0.0) + 2 * (ur > 0.0) + 4 * (ll > 0.0) + 8 * (lr > 0.0);
  if (cs == 0 || cs == 15) return 0;
  const double r1 = r0 + 1.0, c1 = c0 + 1.0;
  const double top_c = __dadd_rn(c0, ms_fraction(ul, ur));
  const double bot_c = __dadd_rn(c0, ms_fraction(ll, lr));
  const double left_r = __dadd_rn(r0, ms_fraction(ul, ll));
  const double right_r = __dadd_rn(r0, ms_fraction(ur, lr));
  // edge points: T(r0, top_c)  B(r1, bot_c)  L(left_r, c0)  R(right_r, c1)
  enum { T, B, L, R };
  int a0 = -1, b0 = -1, a1 = -1, b1 = -1;
  switch (cs) {
    case 1: a0 = T; b0 = L; break;
    case 2: a0 = R; b0 = T; break;
    case 3: a0 = R; b0 = L; break;
    case 4: a0 = L; b0 = B; break;
    case 5: a0 = T; b0 = B; break;
    case 6: a0 = R; b0 = T; a1 = L; b1 = B; break;      // low values connected
    case 7: a0 = R; b0 = B; break;
    case 8: a0 = B; b0 = R; break;
    case 9: a0 = T; b0 = L; a1 = B; b1 = R; break;      // low values connected
    case 10: a0 = B; b0 = T; break;
    case 11: a0 = B; b0 = L; break;
    case 12: a0 = L; b0 = R; break;
    case 13: a0 = T; b0 = R; break;
    case 14: a0 = L; b0 = T; break;
  }
  // register selects (no local-memory arrays)
  auto prow = [&](int k) { return k == T ? r0 : k == B ? r1 : k == L ? left_r : right_r; };
  auto pcol = [&](int k) { return k == T ? top_c : k == B ? bot_c : k == L ? c0 : c1; };
  int n = 0;
  {
    const double fr = prow(a0), fc = pcol(a0), tr = prow(b0), tc = pcol(b0);
    if (fr != tr || fc != tc) {
      if (out) out[n] = Seg{fr, fc, tr, tc};
      ++n;
    }
  }
  if (a1 >= 0) {
    const double fr = prow(a1), fc = pcol(a1), tr = prow(b1), tc = pcol(b1);
    if (fr != tr || fc != tc) {
      if (out) out[n] = Seg{fr, fc, tr, tc};
      ++n;
    }
  }
  return n;
}

// Block-wide exclusive scan of one int per thread; returns the block total.
__device__ __forceinline__ int block_exclusive_scan(int v, int* excl, int* s_warp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int w = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) s_warp[lane] = w;       // inclusive warp totals
  }
  __syncthreads();
  const int total = s_warp[(blockDim.x >> 5) - 1];
  *excl = x - v + (wid ? s_warp[wid - 1] : 0);
  __syncthreads();
  return total;
}

// One CTA per square row (grid max(H - 1, 1)).  COUNT: segments per square
// row -> cnt[r0], and the field's sign flags (bit 0: some phi > 0, bit 1:
// some phi < 0) over pixel rows r0 (and H - 1 for the last CTA).  WRITE:
// the row's segments in square order at off[r0].
template <bool WRITE>
__global__ void __launch_bounds__(kContourThreads)
k_contour_rows(const double* __restrict__ phi, long long H, long long W,
               long long* __restrict__ cnt, const long long* __restrict__ off,
               Seg* __restrict__ segs, unsigned* __restrict__ signs) {
  __shared__ int s_warp[kContourThreads / 32];
  const long long r0 = blockIdx.x;
  if (!WRITE) {
    unsigned f = 0;
    const long long rlast = (r0 == gridDim.x - 1) ? H - 1 : r0;
    for (long long r = r0; r <= rlast; ++r)
      for (long long c = threadIdx.x; c < W; c += blockDim.x) {
        const double v = phi[r * W + c];
        f |= (v > 0.0) ? 1u : 0u;
        f |= (v < 0.0) ? 2u : 0u;
      }
    f = __reduce_or_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(signs, f);
  }
  if (r0 + 1 >= H) {
    if (!WRITE && threadIdx.x == 0) cnt[r0] = 0;
    return;
  }
  const double* a = phi + r0 * W;
  const double* b = a + W;
  long long base = WRITE ? off[r0] : 0;
  long long total = 0;
  for (long long c0 = 0; c0 < W - 1; c0 += blockDim.x) {
    const long long c = c0 + threadIdx.x;
    Seg s[2];
    int n = 0;
    if (c < W - 1)
      n = ms_square(a[c], a[c + 1], b[c], b[c + 1], (double)r0, (double)c, WRITE ? s : nullptr);
    if (WRITE) {
      int ex;
      const int t = block_exclusive_scan(n, &ex, s_warp);
      for (int k = 0; k < n; ++k) segs[base + ex + k] = s[k];
      base += t;
    } else {
      total += n;
    }
  }
  if (!WRITE) {
    total = __reduce_add_sync(0xffffffffu, (unsigned)total);   // <= 2 W per row
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = (int)total;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_warp[w];
      cnt[r0] = t;
    }
  }
}

// Exclusive scan of the per-row counts (one CTA, n rows); off[n] = total.
__global__ void __launch_bounds__(1024) k_contour_scan(const long long* __restrict__ cnt,
                                                       long long n,
                                                       long long* __restrict__ off) {
  __shared__ long long s[1024];
  const long long per = (n + blockDim.x - 1) / blockDim.x;
  const long long lo = threadIdx.x * per, hi = lo + per < n ? lo + per : n;
  long long t = 0;
  for (long long i = lo; i < hi; ++i) t += cnt[i];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const long long y = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += y;
    __syncthreads();
  }
  long long run = s[threadIdx.x] - t;
  for (long long i = lo; i < hi; ++i) {
    off[i] = run;
    run += cnt[i];
  }
  if (threadIdx.x == blockDim.x - 1) off[n] = s[threadIdx.x];
}

// ------------------------------------------------------------- host assembly
struct MsPoint {
  double r, c;
  bool operator==(const MsPoint& o) const { return r == o.r && c == o.c; }
};

struct MsPointHash {
  size_t operator()(const MsPoint& p) const {
    uint64_t a, b;
    const double r = p.r + 0.0, c = p.c + 0.0;     // -0.0 hashes as +0.0
    memcpy(&a, &r, 8);
    memcpy(&b, &c, 8);
    uint64_t h = a * 0x9E3779B97F4A7C15ull;
    h ^= b + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
    return (size_t)(h ^ (h >> 31));
  }
};

// Joins segments (in square order) into polylines; returns them in creation
// order as (row, col) points.  Mirrors the dict semantics of the published
// assembly: pop-and-reinsert on starts / ends, the earlier-created contour
// survives a join, a join of a contour with itself closes it.
inline std::vector<std::deque<MsPoint>> ms_assemble(const std::vector<Seg>& segs) {
  std::vector<std::deque<MsPoint>> contours;
  std::vector<char> alive;
  std::unordered_map<MsPoint, long long, MsPointHash> starts, ends;
  starts.reserve(segs.size() / 4 + 16);
  ends.reserve(segs.size() / 4 + 16);
  auto pop = [](std::unordered_map<MsPoint, long long, MsPointHash>& m, const MsPoint& k) {
    auto it = m.find(k);
    if (it == m.end()) return -1LL;
    const long long v = it->second;
    m.erase(it);
    return v;
  };
  for (const Seg& s : segs) {
    const MsPoint from{s.fr, s.fc}, to{s.tr, s.tc};
    if (from == to) continue;
    const long long tail = pop(starts, to);
    const long long head = pop(ends, from);
    if (tail >= 0 && head >= 0) {
      if (tail == head) {
        contours[head].push_back(to);                 // closes the contour
      } else if (tail > head) {                       // tail created later: append it to head
        auto& H = contours[head];
        auto& T = contours[tail];
        H.insert(H.end(), T.begin(), T.end());
        T.clear();
        alive[tail] = 0;
        starts[H.front()] = head;
        ends[H.back()] = head;
      } else {                                        // head created later: prepend it to tail
        auto& H = contours[head];
        auto& T = contours[tail];
        T.insert(T.begin(), H.begin(), H.end());
        pop(starts, H.front());
        H.clear();
        alive[head] = 0;
        starts[T.front()] = tail;
        ends[T.back()] = tail;
      }
    } else if (tail < 0 && head < 0) {
      const long long id = (long long)contours.size();
      contours.emplace_back(std::deque<MsPoint>{from, to});
      alive.push_back(1);
      starts[from] = id;
      ends[to] = id;
    } else if (head < 0) {                            // segment precedes tail
      contours[tail].push_front(from);
      starts[from] = tail;
    } else {                                          // segment follows head
      contours[head].push_back(to);
      ends[to] = head;
    }
  }
  std::vector<std::deque<MsPoint>> out;
  for (size_t i = 0; i < contours.size(); ++i)
    if (alive[i]) out.push_back(std::move(contours[i]));
  return out;
}

}  // namespace lse
