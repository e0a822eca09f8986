// mba_match.cu -- batched descriptor matching: frontend.match
// (frontend.py:220-250) for every listed frame pair in one call -- the
// exhaustive pairwise matching that build_tracks (miniba.py:555-591) runs
// before its union-find.
//
// Per pair (A, B): 256-bit Hamming distances (8 x popc of XOR), for every row
// a the nearest b (first index on ties) and the second-smallest distance
// (duplicates counted, as np.partition), the ratio test best/second <
// ratio_max (ratio 1 when second == 0; always passed when |B| < 2); the same
// per column; a match is mutual and passes both ratio tests. Integer
// distances -> results identical to the reference.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mba_common.cuh"

namespace mba {

constexpr int kMatchThreads = 128;
constexpr int kDescWords = 8;   // 256 bits

// One thread per query descriptor of frame `q`, scanning every descriptor of
// frame `r` (staged in shared memory in tiles).
__global__ void __launch_bounds__(kMatchThreads) nn_kernel(
    const uint32_t* __restrict__ desc, const int64_t* __restrict__ off, const int32_t* __restrict__ pairs,
    int swap, const int64_t* __restrict__ row_off, int n_pairs, double ratio_max, int32_t* __restrict__ nn_out,
    uint8_t* __restrict__ ok_out, int32_t* __restrict__ best_out) {
  __shared__ uint32_t tile[kMatchThreads][kDescWords + 1];
  const int p = blockIdx.y;
  if (p >= n_pairs) return;
  const int fq = pairs[2 * p + (swap ? 1 : 0)], fr = pairs[2 * p + (swap ? 0 : 1)];
  const int64_t q0 = off[fq], nq = off[fq + 1] - q0, r0 = off[fr], nr = off[fr + 1] - r0;
  const int64_t qi = (int64_t)blockIdx.x * kMatchThreads + threadIdx.x;
  if ((int64_t)blockIdx.x * kMatchThreads >= nq) return;   // uniform per block
  uint32_t me[kDescWords];
  if (qi < nq)
#pragma unroll
    for (int w = 0; w < kDescWords; ++w) me[w] = __ldg(desc + (q0 + qi) * kDescWords + w);
  int best = 1 << 30, second = 1 << 30, nn = 0;
  for (int64_t t0 = 0; t0 < nr; t0 += kMatchThreads) {
    __syncthreads();
    if (t0 + threadIdx.x < nr)
#pragma unroll
      for (int w = 0; w < kDescWords; ++w) tile[threadIdx.x][w] = __ldg(desc + (r0 + t0 + threadIdx.x) * kDescWords + w);
    __syncthreads();
    const int cnt = (int)(nr - t0 < kMatchThreads ? nr - t0 : kMatchThreads);
    if (qi < nq)
      for (int j = 0; j < cnt; ++j) {
        int d = 0;
#pragma unroll
        for (int w = 0; w < kDescWords; ++w) d += __popc(me[w] ^ tile[j][w]);
        if (d < best) {
          second = best;
          best = d;
          nn = (int)(t0 + j);
        } else if (d < second) {
          second = d;
        }
      }
  }
  if (qi >= nq) return;
  bool ok = true;
  if (nr == 0) {   // empty frame: no match (frontend.py:225-227)
    nn = -1;
    ok = false;
  } else if (nr >= 2) {
    const double ratio = second > 0 ? (double)best / (double)second : 1.0;
    ok = ratio < ratio_max;
  }
  const int64_t o = row_off[p] + qi;
  nn_out[o] = nn;
  ok_out[o] = ok ? 1 : 0;
  if (best_out) best_out[o] = best;
}

// mutual check per row of A: match_b[a] = b (or -1), dist[a]
__global__ void mutual_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ pairs,
                              const int64_t* __restrict__ row_a, const int64_t* __restrict__ row_b,
                              int n_pairs, const int32_t* __restrict__ nn_ab, const uint8_t* __restrict__ ok_a,
                              const int32_t* __restrict__ best_ab, const int32_t* __restrict__ nn_ba,
                              const uint8_t* __restrict__ ok_b, int32_t* __restrict__ match_b,
                              int32_t* __restrict__ dist) {
  const int p = blockIdx.y;
  if (p >= n_pairs) return;
  const int fa = pairs[2 * p];
  const int64_t na = off[fa + 1] - off[fa];
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const int64_t o = row_a[p] + a;
  const int b = nn_ab[o];
  const bool m = b >= 0 && ok_a[o] && nn_ba[row_b[p] + b] == a && ok_b[row_b[p] + b];
  match_b[o] = m ? b : -1;
  dist[o] = best_ab[o];
}

}  // namespace mba

extern "C" int32_t mba_match_pairs(int32_t n_frames, const uint8_t* desc, const int64_t* desc_off,
                                   int32_t n_pairs, const int32_t* pairs, const int64_t* row_off_a,
                                   const int64_t* row_off_b, int64_t max_rows, double ratio_max,
                                   int32_t* nn_ab, uint8_t* ok_a, int32_t* best_ab, int32_t* nn_ba,
                                   uint8_t* ok_b, int32_t* match_b, int32_t* dist, void* stream) {
  if (n_frames < 0 || n_pairs < 0 || max_rows < 0) return MBA_ERR_INVALID;
  if (n_pairs == 0 || max_rows == 0) return MBA_OK;
  if (!desc || !desc_off || !pairs || !row_off_a || !row_off_b || !nn_ab || !ok_a || !best_ab || !nn_ba ||
      !ok_b || !match_b || !dist)
    return MBA_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned gx = (unsigned)((max_rows + mba::kMatchThreads - 1) / mba::kMatchThreads);
  const dim3 grid(gx, (unsigned)n_pairs);
  const uint32_t* d32 = reinterpret_cast<const uint32_t*>(desc);
  mba::nn_kernel<<<grid, mba::kMatchThreads, 0, st>>>(d32, desc_off, pairs, 0, row_off_a, n_pairs, ratio_max,
                                                      nn_ab, ok_a, best_ab);
  mba::nn_kernel<<<grid, mba::kMatchThreads, 0, st>>>(d32, desc_off, pairs, 1, row_off_b, n_pairs, ratio_max,
                                                      nn_ba, ok_b, nullptr);
  mba::mutual_kernel<<<grid, mba::kMatchThreads, 0, st>>>(desc_off, pairs, row_off_a, row_off_b, n_pairs,
                                                          nn_ab, ok_a, best_ab, nn_ba, ok_b, match_b, dist);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}
