// Word-set tables on device (north_star subsystem 1).
//
// Restates, bit for bit, the reference's host-side table construction:
//   letters        wordsets.py:176-188   (code // d^(n-1-j)) % d, zero padded
//   prefix/suffix  wordsets.py:190-228   position of code // d^(n-k) (prefix) or
//                                        code % d^k (suffix) among the length-k
//                                        words, EPSILON_INDEX (-1) at k = 0,
//                                        MISSING_INDEX (-2) if absent or k > n
//   level starts   wordsets.py:230-247   start of each length block
//   packed letters words.py:158-174      letter j at bits b*j, b = bits_per_letter
// The dict lookup of the reference (global_index) becomes a binary search of
// the canonical (length asc, code asc) order inside the level block, which is
// the same map because the order is strict.  Integer work only.
#include "sigb_internal.h"

namespace sigb {
namespace {

constexpr int64_t kEpsilon = -1;
constexpr int64_t kMissing = -2;

__device__ __forceinline__ uint64_t upow(uint64_t d, int64_t e) {
  uint64_t p = 1;
  for (int64_t i = 0; i < e; ++i) p *= d;
  return p;
}

// level_start[n] = number of words shorter than n (lower bound of n).
__global__ void level_start_kernel(const int64_t* __restrict__ lengths, int64_t W, int64_t max_len,
                                   int64_t* __restrict__ level_start) {
  int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n > max_len + 1) return;
  int64_t lo = 0, hi = W;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (lengths[mid] < n) lo = mid + 1; else hi = mid;
  }
  level_start[n] = lo;
}

__device__ __forceinline__ int64_t find_in_level(const uint64_t* __restrict__ codes,
                                                 const int64_t* __restrict__ level_start,
                                                 int64_t k, uint64_t code) {
  int64_t lo = level_start[k], hi = level_start[k + 1];
  const int64_t end = hi;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (codes[mid] < code) lo = mid + 1; else hi = mid;
  }
  return (lo < end && codes[lo] == code) ? lo : kMissing;
}

// One thread per word: its letters, packed letters and both factor tables.
__global__ void tables_kernel(const uint64_t* __restrict__ codes, const int64_t* __restrict__ lengths,
                              int64_t W, int64_t d, int64_t max_len, int bits,
                              const int64_t* __restrict__ level_start, int64_t* __restrict__ letters,
                              int64_t* __restrict__ prefix, int64_t* __restrict__ suffix,
                              uint64_t* __restrict__ packed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= W) return;
  const uint64_t code = codes[i];
  const int64_t n = lengths[i];
  const uint64_t ud = (uint64_t)d;
  uint64_t pk = 0;
  // letters[i, j] for j < n, most significant digit first
  {
    uint64_t rem = code;
    for (int64_t j = n - 1; j >= 0; --j) {
      uint64_t l = rem % ud;
      rem /= ud;
      if (letters) letters[i * max_len + j] = (int64_t)l;
      if (packed) pk |= l << (uint64_t)(bits * j);
    }
    if (letters)
      for (int64_t j = n; j < max_len; ++j) letters[i * max_len + j] = 0;
  }
  if (packed) packed[i] = pk;
  const int64_t C = max_len + 1;
  if (prefix) prefix[i * C] = kEpsilon;
  if (suffix) suffix[i * C] = kEpsilon;
  for (int64_t k = 1; k < C; ++k) {
    if (k > n) {
      if (prefix) prefix[i * C + k] = kMissing;
      if (suffix) suffix[i * C + k] = kMissing;
      continue;
    }
    if (prefix) prefix[i * C + k] = find_in_level(codes, level_start, k, code / upow(ud, n - k));
    if (suffix) {
      // code % d^n == code (and d^n may be 2^64, which wraps): special-case k == n
      uint64_t sub = (k == n) ? code : code % upow(ud, k);
      suffix[i * C + k] = find_in_level(codes, level_start, k, sub);
    }
  }
}

}  // namespace

int launch_wordset_tables(const uint64_t* d_codes, const int64_t* d_lengths, int64_t W, int64_t d,
                          int64_t max_len, int64_t* d_letters, int64_t* d_prefix, int64_t* d_suffix,
                          int64_t* d_level_start, uint64_t* d_packed, cudaStream_t stream) {
  if (W < 0 || d < 1 || max_len < 0) return fail(SIGB_ERR_DOMAIN, "invalid word-set dimensions");
  if (d_level_start == nullptr) return fail(SIGB_ERR_DOMAIN, "level_start output is required");
  int bits = 1;
  while ((int64_t(1) << bits) < d) ++bits;
  if (d_packed && bits * max_len > 64)
    return fail(SIGB_ERR_CAPACITY, std::to_string(max_len) + " letters at " + std::to_string(bits) +
                                       " bits each exceed 64 bits");
  level_start_kernel<<<(unsigned)((max_len + 2 + 127) / 128), 128, 0, stream>>>(d_lengths, W, max_len,
                                                                                d_level_start);
  SIGB_CUDA_TRY(cudaGetLastError());
  if (W > 0) {
    tables_kernel<<<(unsigned)((W + 255) / 256), 256, 0, stream>>>(
        d_codes, d_lengths, W, d, max_len, bits, d_level_start, d_letters, d_prefix, d_suffix, d_packed);
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}

}  // namespace sigb
