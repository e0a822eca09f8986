// mba_match.cu -- batched descriptor matching: frontend.match
// (frontend.py:220-250) for every listed frame pair in one call -- the
// exhaustive pairwise matching that build_tracks (miniba.py:555-591) runs
// before its union-find.
//
// Semantics per pair (A, B): 256-bit Hamming distances; for every row a the
// nearest b (first index on ties) and the second-smallest distance
// (duplicates counted, as np.partition), the ratio test best/second <
// ratio_max (ratio 1 when second == 0; always passed when |B| < 2); the same
// per column; a match is mutual and passes both ratio tests. Integer
// distances -> results identical to the reference.
//
// Every distance is computed ONCE: a CTA owns a 64 x 64 tile (rows of A x
// columns of B) of one pair, stages both descriptor tiles in shared memory,
// writes the tile's distances into shared memory (8 x popc of XOR each) and
// reduces them row-wise and column-wise into per-tile partials (best,
// second, argmin). A second kernel merges the partials of each row across the
// column tiles (and of each column across the row tiles) in tile order --
// the earlier tile wins ties, which keeps "first index on ties" -- and a third
// applies the ratio tests and the mutual check.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mba_common.cuh"

namespace mba {
namespace match {

constexpr int kTile = 64;
constexpr int kWords = 8;   // 256 bits

struct Part {
  int best, second, nn;
};

// merge b (from a LATER tile) into a (earlier tile): strict < keeps the
// earlier index on ties; second counts duplicates
__device__ __forceinline__ Part merge(Part a, Part b) {
  Part o;
  if (b.best < a.best) {
    o.best = b.best;
    o.nn = b.nn;
    o.second = min(a.best, b.second);
  } else {
    o.best = a.best;
    o.nn = a.nn;
    o.second = min(a.second, b.best);
  }
  return o;
}

// grid: (tiles of A rows, tiles of B cols, pair). Partials:
//   row_part[row_off_a[p] + a][tb] and col_part[row_off_b[p] + b][ta]
__global__ void __launch_bounds__(kTile * 4) tile_kernel(const uint32_t* __restrict__ desc,
                                                          const int64_t* __restrict__ off,
                                                          const int32_t* __restrict__ pairs,
                                                          const int64_t* __restrict__ row_a,
                                                          const int64_t* __restrict__ row_b, int n_tiles_b_max,
                                                          int n_tiles_a_max, int4* __restrict__ row_part,
                                                          int4* __restrict__ col_part) {
  __shared__ uint32_t sa[kTile][kWords + 1], sb[kTile][kWords + 1];
  __shared__ unsigned short dist[kTile][kTile + 1];
  const int p = blockIdx.z;
  const int fa = pairs[2 * p], fb = pairs[2 * p + 1];
  const int64_t a0 = off[fa], na = off[fa + 1] - a0, b0 = off[fb], nb = off[fb + 1] - b0;
  const int ta = blockIdx.x, tb = blockIdx.y;
  if ((int64_t)ta * kTile >= na || (int64_t)tb * kTile >= nb) return;   // uniform per block
  const int tid = threadIdx.x;
  for (int i = tid; i < kTile * kWords; i += blockDim.x) {
    const int r = i / kWords, w = i % kWords;
    const int64_t ra = (int64_t)ta * kTile + r, rb = (int64_t)tb * kTile + r;
    sa[r][w] = ra < na ? __ldg(desc + (a0 + ra) * kWords + w) : 0u;
    sb[r][w] = rb < nb ? __ldg(desc + (b0 + rb) * kWords + w) : 0u;
  }
  __syncthreads();
  // the tile's distances, each computed once: a 4 x 4 register block per
  // thread (4 rows of A and 4 columns of B held in registers, 4 shared loads
  // per distance instead of 16)
  for (int blk = tid; blk < (kTile / 4) * (kTile / 4); blk += blockDim.x) {
    const int r0 = (blk / (kTile / 4)) * 4, c0 = (blk % (kTile / 4)) * 4;
    int d[4][4] = {};
#pragma unroll
    for (int w = 0; w < kWords; ++w) {
      uint32_t a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = sa[r0 + q][w];
        b[q] = sb[c0 + q][w];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) d[i][j] += __popc(a[i] ^ b[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dist[r0 + i][c0 + j] = (unsigned short)d[i][j];
  }
  __syncthreads();
  const int64_t ra_left = na - (int64_t)ta * kTile, rb_left = nb - (int64_t)tb * kTile;
  const int nr = ra_left < kTile ? (int)ra_left : kTile;
  const int nc = rb_left < kTile ? (int)rb_left : kTile;
  if (tid < kTile) {   // row partials
    const int r = tid;
    if (r < nr) {
      Part q{1 << 30, 1 << 30, 0};
      for (int c = 0; c < nc; ++c) {
        const int d = dist[r][c];
        if (d < q.best) {
          q.second = q.best;
          q.best = d;
          q.nn = tb * kTile + c;
        } else if (d < q.second) {
          q.second = d;
        }
      }
      row_part[(row_a[p] + (int64_t)ta * kTile + r) * n_tiles_b_max + tb] = make_int4(q.best, q.second, q.nn, 0);
    }
  } else if (tid < 2 * kTile) {   // column partials
    const int c = tid - kTile;
    if (c < nc) {
      Part q{1 << 30, 1 << 30, 0};
      for (int r = 0; r < nr; ++r) {
        const int d = dist[r][c];
        if (d < q.best) {
          q.second = q.best;
          q.best = d;
          q.nn = ta * kTile + r;
        } else if (d < q.second) {
          q.second = d;
        }
      }
      col_part[(row_b[p] + (int64_t)tb * kTile + c) * n_tiles_a_max + ta] = make_int4(q.best, q.second, q.nn, 0);
    }
  }
}

// merge the partials of one row (or column) in tile order; ratio test
__global__ void reduce_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ pairs, int side,
                              const int64_t* __restrict__ rows, int n_pairs, int n_tiles_max,
                              const int4* __restrict__ part, double ratio_max, int32_t* __restrict__ nn_out,
                              uint8_t* __restrict__ ok_out, int32_t* __restrict__ best_out) {
  const int p = blockIdx.y;
  if (p >= n_pairs) return;
  const int f = pairs[2 * p + side], g = pairs[2 * p + 1 - side];
  const int64_t n = off[f + 1] - off[f], m = off[g + 1] - off[g];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t o = rows[p] + i;
  const int nt = (int)((m + kTile - 1) / kTile);
  int nn = -1;
  bool ok = false;
  int best = 1 << 30;
  if (nt > 0) {
    const int4 v0 = part[o * n_tiles_max];
    Part q{v0.x, v0.y, v0.z};
    for (int t = 1; t < nt; ++t) {
      const int4 v = part[o * n_tiles_max + t];
      q = merge(q, Part{v.x, v.y, v.z});
    }
    nn = q.nn;
    best = q.best;
    ok = true;
    if (m >= 2) {
      const double ratio = q.second > 0 ? (double)q.best / (double)q.second : 1.0;
      ok = ratio < ratio_max;
    }
  }
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

}  // namespace match
}  // namespace mba

extern "C" size_t mba_match_workspace_bytes(int64_t rows_a, int64_t rows_b, int64_t max_rows) {
  const int64_t nt = (max_rows + mba::match::kTile - 1) / mba::match::kTile;
  return (size_t)(rows_a + rows_b) * (size_t)(nt > 0 ? nt : 1) * sizeof(int4);
}

extern "C" int32_t mba_match_pairs(int32_t n_frames, const uint8_t* desc, const int64_t* desc_off,
                                   int32_t n_pairs, const int32_t* pairs, const int64_t* row_off_a,
                                   const int64_t* row_off_b, int64_t max_rows, double ratio_max,
                                   int32_t* nn_ab, uint8_t* ok_a, int32_t* best_ab, int32_t* nn_ba,
                                   uint8_t* ok_b, int32_t* match_b, int32_t* dist, int64_t rows_a,
                                   int64_t rows_b, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace mba::match;
  if (n_frames < 0 || n_pairs < 0 || max_rows < 0) return MBA_ERR_INVALID;
  if (n_pairs == 0 || max_rows == 0) return MBA_OK;
  if (!desc || !desc_off || !pairs || !row_off_a || !row_off_b || !nn_ab || !ok_a || !best_ab || !nn_ba ||
      !ok_b || !match_b || !dist || !workspace)
    return MBA_ERR_INVALID;
  if (workspace_bytes < mba_match_workspace_bytes(rows_a, rows_b, max_rows)) return MBA_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const int nt = (int)((max_rows + kTile - 1) / kTile);
  int4* row_part = (int4*)workspace;
  int4* col_part = row_part + (size_t)rows_a * nt;
  const uint32_t* d32 = reinterpret_cast<const uint32_t*>(desc);
  tile_kernel<<<dim3(nt, nt, n_pairs), kTile * 4, 0, st>>>(d32, desc_off, pairs, row_off_a, row_off_b, nt, nt,
                                                           row_part, col_part);
  const unsigned gx = (unsigned)((max_rows + 127) / 128);
  reduce_kernel<<<dim3(gx, n_pairs), 128, 0, st>>>(desc_off, pairs, 0, row_off_a, n_pairs, nt, row_part,
                                                   ratio_max, nn_ab, ok_a, best_ab);
  reduce_kernel<<<dim3(gx, n_pairs), 128, 0, st>>>(desc_off, pairs, 1, row_off_b, n_pairs, nt, col_part,
                                                   ratio_max, nn_ba, ok_b, nullptr);
  mutual_kernel<<<dim3(gx, n_pairs), 128, 0, st>>>(desc_off, pairs, row_off_a, row_off_b, n_pairs, nn_ab, ok_a,
                                                   best_ab, nn_ba, ok_b, match_b, dist);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}
