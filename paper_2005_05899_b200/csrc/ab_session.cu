// C-ABI session: ab_ctx_create / ab_mesh_upload / ab_state_set / ab_step /
// ab_state_get / ab_ctx_destroy (include/alyab200.h "Session", SURVEY.md
// §8(b)(3)).  A C, C++ or FFI caller hands over host arrays once (nodes,
// per-category connectivity, boundary data) and then advances the solution
// with one call per time step; every setup structure the Python layer builds
// (device.py: SFC element order, node windows; solver.py: CSR pattern,
// Laplacian, SELL-32, gradient operator, SFC row order of the pressure
// system) is built here by device code (sort/scan/unique on the GPU, the
// library's own assembly kernels), and ab_step launches exactly the kernel
// sequence of FlowSolver._step_body (Algorithm 1).
//
// Setup choices that only change rounding (the bank-aware tet node order and
// the bank-spread reference order of device.py) are not applied here; the
// pressure solve is the tiled single-pass CG on D^-1/2 P L P^T D^-1/2 in the Hilbert order (two-kernel Jacobi-PCG on P L P^T if a tile map does not fit 16 bits)
// of the nodes (the path of every system too large for the on-chip solver).
#include <thrust/binary_search.h>
#include <thrust/copy.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <thrust/reduce.h>
#include <thrust/scan.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>
#include <thrust/transform_reduce.h>
#include <thrust/unique.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "ab_common.cuh"

namespace ab {
namespace {

constexpr int kWinBlock = 128;
constexpr int kNodeNN[5] = {4, 4, 5, 6, 8};  // AB_RULE_* -> nodes per element

__global__ void k_expand34(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  b[4 * i] = a[3 * i];
  b[4 * i + 1] = a[3 * i + 1];
  b[4 * i + 2] = a[3 * i + 2];
  b[4 * i + 3] = 0.0;
}
__global__ void k_compact43(int64_t n, const double* __restrict__ b, double* __restrict__ a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  a[3 * i] = b[4 * i];
  a[3 * i + 1] = b[4 * i + 1];
  a[3 * i + 2] = b[4 * i + 2];
}
__global__ void k_coords3(int64_t n, const double* __restrict__ c4, double* __restrict__ c3) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { c3[3 * i] = c4[4 * i]; c3[3 * i + 1] = c4[4 * i + 1]; c3[3 * i + 2] = c4[4 * i + 2]; }
}
__global__ void k_gather_rows(int64_t e, int nn, const int32_t* __restrict__ in, const int64_t* __restrict__ order,
                              int32_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= e * nn) return;
  const int64_t r = t / nn;
  out[t] = in[order[r] * nn + (t - r * nn)];
}
__global__ void k_iota64(int64_t n, int64_t* __restrict__ a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}
// window keys: (block, node) of every element-node reference r = e * nn + a
__global__ void k_win_keys(int64_t e, int nn, const int32_t* __restrict__ conn, int64_t n_nodes,
                           int64_t* __restrict__ keys, int64_t* __restrict__ ref) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= e * nn) return;
  keys[r] = (r / nn / kWinBlock) * n_nodes + conn[r];
  ref[r] = r;
}
__global__ void k_run_flags(int64_t m, const int64_t* __restrict__ ks, int64_t* __restrict__ f) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) f[i] = (i == 0 || ks[i] != ks[i - 1]) ? 1 : 0;
}
// per sorted reference i (uid = window node index, global): window arrays
__global__ void k_win_fill(int64_t m, int nn, int64_t n_nodes, const int64_t* __restrict__ ks,
                           const int64_t* __restrict__ ref, const int64_t* __restrict__ uid1,
                           int32_t* __restrict__ wnode, int32_t* __restrict__ wptr, int64_t* __restrict__ wblk,
                           uint16_t* __restrict__ wslot) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t u = uid1[i] - 1;
  if (i == 0 || ks[i] != ks[i - 1]) {
    wnode[u] = (int32_t)(ks[i] % n_nodes);
    wblk[u] = ks[i] / n_nodes;
    wptr[u] = (int32_t)i;
  }
  const int64_t r = ref[i];
  const int64_t e = r / nn;
  const int a = (int)(r - e * nn);
  wslot[i] = (uint16_t)(a * kWinBlock + (int)(e % kWinBlock));
}
__global__ void k_win_local(int64_t m, int nn, const int64_t* __restrict__ ref, const int64_t* __restrict__ uid1,
                            const int64_t* __restrict__ blk_ptr, const uint16_t* __restrict__ wslot,
                            uint16_t* __restrict__ loc, uint32_t* __restrict__ wref) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t r = ref[i];
  const int64_t b = r / nn / kWinBlock;
  const int64_t local = uid1[i] - 1 - blk_ptr[b];
  loc[r] = (uint16_t)local;
  wref[i] = (uint32_t)wslot[i] | ((uint32_t)local << 16);
}
__global__ void k_win_desc(int64_t nblk, const int64_t* __restrict__ blk_ptr, const int32_t* __restrict__ wptr,
                           int32_t* __restrict__ desc) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const int64_t b0 = blk_ptr[b], b1 = blk_ptr[b + 1];
  desc[4 * b] = (int32_t)b0;
  desc[4 * b + 1] = (int32_t)b1;
  desc[4 * b + 2] = wptr[b0];
  desc[4 * b + 3] = wptr[b1];
}
__global__ void k_fill_u32(int64_t n, uint32_t v, uint32_t* __restrict__ a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
// (row, col) keys of every element node pair
__global__ void k_pair_keys(int64_t e, int nn, const int32_t* __restrict__ conn, int64_t n_nodes,
                            int64_t* __restrict__ keys) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)nn * nn;
  if (t >= e * per) return;
  const int64_t el = t / per;
  const int ab = (int)(t - el * per);
  const int a = ab / nn, b = ab - a * nn;
  keys[t] = (int64_t)conn[el * nn + a] * n_nodes + conn[el * nn + b];
}
__global__ void k_split_keys(int64_t m, const int64_t* __restrict__ keys, int64_t n_nodes, int64_t* __restrict__ rows,
                             int32_t* __restrict__ cols) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (rows) rows[i] = keys[i] / n_nodes;
  cols[i] = (int32_t)(keys[i] % n_nodes);
}
__global__ void k_row_of(int64_t n, const int64_t* __restrict__ rp, int64_t* __restrict__ row) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) row[k] = i;
}
__global__ void k_perm_keys(int64_t m, const int64_t* __restrict__ row, const int32_t* __restrict__ cols,
                            const int64_t* __restrict__ iperm, int64_t n, int64_t* __restrict__ keys,
                            int64_t* __restrict__ idx) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  keys[k] = iperm[row[k]] * n + iperm[cols[k]];
  idx[k] = k;
}
__global__ void k_gather_f64(int64_t m, const double* __restrict__ a, const int64_t* __restrict__ idx,
                             double* __restrict__ b) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) b[k] = a[idx[k]];
}
__global__ void k_gather_u8(int64_t m, const uint8_t* __restrict__ a, const int64_t* __restrict__ idx,
                            uint8_t* __restrict__ b) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) b[k] = a[idx[k]];
}
__global__ void k_invert(int64_t n, const int64_t* __restrict__ perm, int64_t* __restrict__ iperm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) iperm[perm[i]] = i;
}
__global__ void k_slice_width(int64_t n, const int64_t* __restrict__ rp, int64_t* __restrict__ w32) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ns = (n + 31) / 32;
  if (s >= ns) return;
  int64_t w = 0;
  for (int64_t i = 32 * s; i < 32 * s + 32 && i < n; ++i) w = max(w, rp[i + 1] - rp[i]);
  w32[s] = 32 * w;
}
// Unit-diagonal scaled system for the tiled single-pass CG: per-row count of
// the off-diagonal entries, then their compaction (same order).
__global__ void k_count_offdiag(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                int64_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c = 0;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) c += cols[k] != i;
  cnt[i] = c;
}
__global__ void k_compact_offdiag(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                  const double* __restrict__ v, const int64_t* __restrict__ rp2,
                                  int32_t* __restrict__ cols2, double* __restrict__ v2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t o = rp2[i];
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
    if (cols[k] != i) {
      cols2[o] = cols[k];
      v2[o++] = v[k];
    }
}
__global__ void k_sqrt(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = sqrt(a[i]);
}
// Tile map of a SELL-32 matrix (solver.cg_local_map): row i's entries; an own-
// tile column gets its local index, a remote one a key tile * n + col.
__global__ void k_tile_keys(int64_t n, int64_t R, const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
                            uint16_t* __restrict__ lcol, int64_t* __restrict__ key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = i >> 5, t = i / R, r0 = t * R;
  const int64_t b = sp[s] + (i & 31), w = (sp[s + 1] - sp[s]) >> 5;
  for (int64_t j = 0; j < w; ++j) {
    const int64_t e = b + 32 * j;
    const int64_t c = scol[e];
    if (c >= r0 && c < r0 + R) {
      lcol[e] = (uint16_t)(c - r0);
      key[e] = -1;
    } else {
      key[e] = t * n + c;
    }
  }
}
__global__ void k_tile_ghost_cols(int64_t n, int64_t R, const int64_t* __restrict__ sp, const int64_t* __restrict__ key,
                                  const int64_t* __restrict__ gkeys, int64_t ng, const int32_t* __restrict__ gptr,
                                  uint16_t* __restrict__ lcol) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = i >> 5, t = i / R;
  const int64_t b = sp[s] + (i & 31), w = (sp[s + 1] - sp[s]) >> 5;
  for (int64_t j = 0; j < w; ++j) {
    const int64_t e = b + 32 * j;
    const int64_t k = key[e];
    if (k < 0) continue;
    int64_t lo = 0, hi = ng;  // first gkey >= k (present)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (gkeys[mid] < k) lo = mid + 1; else hi = mid;
    }
    lcol[e] = (uint16_t)(R + (lo - gptr[t]));
  }
}
__global__ void k_ghost_split(int64_t ng, int64_t n, const int64_t* __restrict__ gkeys, int32_t* __restrict__ ghost,
                              int64_t* __restrict__ gtile) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  ghost[g] = (int32_t)(gkeys[g] % n);
  gtile[g] = gkeys[g] / n;
}
struct IsRemote {
  __host__ __device__ bool operator()(int64_t k) const { return k >= 0; }
};

__global__ void k_set_diag_fixed(int64_t n, const uint8_t* __restrict__ fixed, double* __restrict__ d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && fixed[i]) d[i] = 1.0;
}

struct RowStart {
  int64_t n;
  __host__ __device__ int64_t operator()(int64_t i) const { return i * n; }
};

struct MinMax3 {
  double lo[3], hi[3];
};
struct MMInit {
  const double* c;
  int stride;
  __host__ __device__ MinMax3 operator()(int64_t i) const {
    MinMax3 r;
    for (int d = 0; d < 3; ++d) r.lo[d] = r.hi[d] = c[i * stride + d];
    return r;
  }
};
struct MMJoin {
  __host__ __device__ MinMax3 operator()(const MinMax3& a, const MinMax3& b) const {
    MinMax3 r;
    for (int d = 0; d < 3; ++d) {
      r.lo[d] = a.lo[d] < b.lo[d] ? a.lo[d] : b.lo[d];
      r.hi[d] = a.hi[d] > b.hi[d] ? a.hi[d] : b.hi[d];
    }
    return r;
  }
};

}  // namespace
}  // namespace ab

using namespace ab;

struct ab_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  std::vector<void*> mem;
  int64_t n = 0;
  ab_mesh mesh{};
  ab_phys phys{};
  double* coords4 = nullptr;
  int32_t* conn[5] = {};
  double* delta2[5] = {};
  double *ml = nullptr, *minv = nullptr;
  // Laplacian (node order, pattern shared with the gradient operator)
  int64_t* rp = nullptr;
  int32_t* cols = nullptr;
  int64_t nnz = 0;
  ab_sell3 B3{};
  // pressure system in the Hilbert row order
  ab_sell Lp{};
  int64_t* perm = nullptr;
  double* dinv_p = nullptr;
  uint8_t* fixed_p = nullptr;
  double *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr, *xn = nullptr;
  // tiled single-pass CG (ab_cg_tile_*): A' = S P L P^T S without its unit
  // diagonal, 2048-row tile map, (x', p) and (r', q) pairs
  bool tiled = false;
  ab_sell Lu{};
  ab_cg_local tmap{};
  int64_t* iperm = nullptr;
  double *s_p = nullptr, *xp = nullptr, *rq[2] = {nullptr, nullptr};
  double *red = nullptr, *sc = nullptr, *part = nullptr;
  uint32_t* cnt = nullptr;
  // state
  double *U0 = nullptr, *U = nullptr, *R = nullptr, *GP = nullptr, *P = nullptr, *Bv = nullptr, *stage = nullptr;
  // boundary data
  int64_t nbc = 0;
  int32_t* bc_idx = nullptr;
  uint8_t* bc_mask = nullptr;
  double* bc_vals = nullptr;
  ab_wall wall{};
  bool ready = false;

  template <class T>
  T* alloc(int64_t count, int64_t pad_bytes = 64) {
    void* q = nullptr;
    const size_t bytes = (size_t)(count > 0 ? count : 1) * sizeof(T) + (size_t)pad_bytes;
    if (cudaMalloc(&q, bytes) != cudaSuccess) return nullptr;
    cudaMemsetAsync(q, 0, bytes, st);
    mem.push_back(q);
    return reinterpret_cast<T*>(q);
  }
  // release a setup temporary early (stream-ordered: after the work queued so far)
  void release(void* q) {
    if (!q) return;
    for (size_t i = 0; i < mem.size(); ++i)
      if (mem[i] == q) {
        cudaStreamSynchronize(st);
        cudaFree(q);
        mem[i] = mem.back();
        mem.pop_back();
        return;
      }
  }
  ~ab_ctx() {
    for (int k = 0; k < 5; ++k)
      if (conn[k]) {
        ab_set_windows(conn[k], kWinBlock, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0);
        ab_set_filter_width(conn[k], 0, nullptr);
      }
    for (void* q : mem) cudaFree(q);
  }
};

namespace {

#define AB_TRY(expr)                        \
  do {                                      \
    if (int rc_ = (expr)) return rc_;       \
  } while (0)
#define AB_ALLOC(ptr_, type_, count_)                                        \
  do {                                                                       \
    (ptr_) = c->alloc<type_>(count_);                                        \
    if (!(ptr_)) return fail("ab_mesh_upload: device memory exhausted");     \
  } while (0)

inline unsigned g256(int64_t n) { return grid_for(n > 0 ? n : 1, 256); }

// Hilbert order (level 10) of n points c (stride doubles apart), keys in the
// box [lo, lo + span) with span = max(hi - lo, 1e-300) * (1 + 1e-12), exactly
// as device.py: stable sort of the keys.
int hilbert_order(ab_ctx* c, int64_t n, const double* pts3, const MinMax3& mm, int64_t* order) {
  double lo_h[3], span_h[3];
  for (int d = 0; d < 3; ++d) {
    lo_h[d] = mm.lo[d];
    double s = mm.hi[d] - mm.lo[d];
    if (s < 1e-300) s = 1e-300;
    span_h[d] = s * (1.0 + 1e-12);
  }
  double* lo = c->alloc<double>(3);
  double* span = c->alloc<double>(3);
  int64_t* keys = c->alloc<int64_t>(n);
  if (!lo || !span || !keys) return fail("ab_mesh_upload: device memory exhausted");
  cudaMemcpyAsync(lo, lo_h, 24, cudaMemcpyHostToDevice, c->st);
  cudaMemcpyAsync(span, span_h, 24, cudaMemcpyHostToDevice, c->st);
  AB_TRY(ab_hilbert_keys(n, pts3, lo, span, 10, keys, c->st));
  k_iota64<<<g256(n), 256, 0, c->st>>>(n, order);
  thrust::stable_sort_by_key(thrust::cuda::par.on(c->st), keys, keys + n, order);
  return check_launch("hilbert_order");
}

MinMax3 minmax(ab_ctx* c, const double* pts, int64_t n, int stride) {
  MinMax3 init;
  for (int d = 0; d < 3; ++d) { init.lo[d] = 1e308; init.hi[d] = -1e308; }
  return thrust::transform_reduce(thrust::cuda::par.on(c->st), thrust::counting_iterator<int64_t>(0),
                                  thrust::counting_iterator<int64_t>(n), MMInit{pts, stride}, init, MMJoin{});
}

// SELL-32 of a CSR matrix (slice pointers computed here), zero-filled padding.
int to_sell(ab_ctx* c, int64_t n, const int64_t* rp, const int32_t* cols, const double* vals, int64_t** sp_out,
            int32_t** scol_out, double** sval_out, double* diag, int64_t* stored) {
  const int64_t ns = (n + 31) / 32;
  int64_t* sp = c->alloc<int64_t>(ns + 1);
  if (!sp) return fail("ab_mesh_upload: device memory exhausted");
  k_slice_width<<<g256(ns), 256, 0, c->st>>>(n, rp, sp + 1);
  thrust::inclusive_scan(thrust::cuda::par.on(c->st), sp + 1, sp + 1 + ns, sp + 1);
  int64_t total = 0;
  cudaMemcpyAsync(&total, sp + ns, 8, cudaMemcpyDeviceToHost, c->st);
  cudaStreamSynchronize(c->st);
  int32_t* scol = *scol_out ? *scol_out : c->alloc<int32_t>(total);
  double* sval = c->alloc<double>(total);
  if (!scol || !sval) return fail("ab_mesh_upload: device memory exhausted");
  AB_TRY(ab_csr_to_sell(n, rp, cols, vals, sp, scol, sval, diag, c->st));
  *sp_out = sp;
  *scol_out = scol;
  *sval_out = sval;
  if (stored) *stored = total;
  return AB_OK;
}

// Tiled single-pass CG setup (solver.PCG's default large-system form):
// A' = S P L P^T S (S = D^-1/2) without its unit diagonal, its 2048-row tile
// map (16-bit tile-local columns, per-tile ghost rows) and the pair vectors.
// Leaves c->tiled false (the plain two-kernel form runs) when a tile's rows
// and ghosts exceed 16 bits.
constexpr int64_t kTileRows = 2048;
int build_tiled_cg(ab_ctx* c, int64_t n, const int64_t* rp, const int32_t* cols, const double* v, int64_t* iperm) {
  int64_t* cnt = c->alloc<int64_t>(n + 1);
  if (!cnt) return fail("ab_mesh_upload: device memory exhausted");
  k_count_offdiag<<<g256(n), 256, 0, c->st>>>(n, rp, cols, cnt + 1);
  thrust::inclusive_scan(thrust::cuda::par.on(c->st), cnt + 1, cnt + 1 + n, cnt + 1);  // cnt[0] = 0 (alloc zeroes)
  int64_t m = 0;
  cudaMemcpyAsync(&m, cnt + n, 8, cudaMemcpyDeviceToHost, c->st);
  cudaStreamSynchronize(c->st);
  int32_t* cols2 = c->alloc<int32_t>(m);
  double* v2 = c->alloc<double>(m);
  if (!cols2 || !v2) return fail("ab_mesh_upload: device memory exhausted");
  k_compact_offdiag<<<g256(n), 256, 0, c->st>>>(n, rp, cols, v, cnt, cols2, v2);
  int64_t* sp = nullptr;
  int32_t* scol = nullptr;
  double* sv = nullptr;
  int64_t stored = 0;
  AB_TRY(to_sell(c, n, cnt, cols2, v2, &sp, &scol, &sv, nullptr, &stored));
  AB_ALLOC(c->s_p, double, n);
  k_sqrt<<<g256(n), 256, 0, c->st>>>(n, c->dinv_p, c->s_p);
  c->Lu = ab_sell{n, (n + 31) / 32, 0, sp, scol, sv};
  AB_TRY(ab_sell_symscale(&c->Lu, c->s_p, c->st));
  // tile map
  const int64_t R = kTileRows, n_t = (n + R - 1) / R;
  uint16_t* lcol = c->alloc<uint16_t>(stored);
  int64_t* key = c->alloc<int64_t>(stored);
  if (!lcol || !key) return fail("ab_mesh_upload: device memory exhausted");
  k_tile_keys<<<g256(n), 256, 0, c->st>>>(n, R, sp, scol, lcol, key);
  int64_t* gk = c->alloc<int64_t>(stored);
  if (!gk) return fail("ab_mesh_upload: device memory exhausted");
  int64_t* gend = thrust::copy_if(thrust::cuda::par.on(c->st), key, key + stored, gk, IsRemote{});
  int64_t ng = gend - gk;
  thrust::sort(thrust::cuda::par.on(c->st), gk, gk + ng);
  ng = thrust::unique(thrust::cuda::par.on(c->st), gk, gk + ng) - gk;
  int32_t* ghost = c->alloc<int32_t>(ng > 0 ? ng : 1);
  int64_t* gtile = c->alloc<int64_t>(ng > 0 ? ng : 1);
  int64_t* gptr64 = c->alloc<int64_t>(n_t + 1);
  int32_t* gptr = c->alloc<int32_t>(n_t + 1);
  if (!ghost || !gtile || !gptr64 || !gptr) return fail("ab_mesh_upload: device memory exhausted");
  if (ng > 0) k_ghost_split<<<g256(ng), 256, 0, c->st>>>(ng, n, gk, ghost, gtile);
  thrust::lower_bound(thrust::cuda::par.on(c->st), gtile, gtile + ng, thrust::counting_iterator<int64_t>(0),
                      thrust::counting_iterator<int64_t>(n_t + 1), gptr64);
  thrust::copy(thrust::cuda::par.on(c->st), gptr64, gptr64 + n_t + 1, gptr);
  std::vector<int64_t> hp(n_t + 1);
  cudaMemcpyAsync(hp.data(), gptr64, 8 * (n_t + 1), cudaMemcpyDeviceToHost, c->st);
  cudaStreamSynchronize(c->st);
  int64_t max_ghost = 0;
  for (int64_t t = 0; t < n_t; ++t) max_ghost = hp[t + 1] - hp[t] > max_ghost ? hp[t + 1] - hp[t] : max_ghost;
  if (R + max_ghost > 65536) {  // stays on the plain two-kernel form
    for (void* q : {(void*)cnt, (void*)cols2, (void*)v2, (void*)key, (void*)gk, (void*)gtile, (void*)gptr64})
      c->release(q);
    return check_launch("ab_mesh_upload");
  }
  k_tile_ghost_cols<<<g256(n), 256, 0, c->st>>>(n, R, sp, key, gk, ng, gptr, lcol);
  // setup temporaries (the CSR copy went into the SELL; keys and ghost tiles are consumed)
  for (void* q : {(void*)cnt, (void*)cols2, (void*)v2, (void*)key, (void*)gk, (void*)gtile, (void*)gptr64}) c->release(q);
  c->tmap = ab_cg_local{};
  c->tmap.rows_per_cta = R;
  c->tmap.n_cta = (int32_t)n_t;
  c->tmap.max_ghost = (int32_t)max_ghost;
  c->tmap.cols = lcol;
  c->tmap.ghost_ptr = gptr;
  c->tmap.ghost = ghost;
  AB_ALLOC(c->xp, double, 2 * n);
  AB_ALLOC(c->rq[0], double, 2 * n);
  AB_ALLOC(c->rq[1], double, 2 * n);
  c->iperm = iperm;
  c->tiled = true;
  return check_launch("ab_mesh_upload");
}

int build_windows(ab_ctx* c, int k, int64_t ne, int nn) {
  const int64_t m = ne * nn;
  const int64_t nblk = (ne + kWinBlock - 1) / kWinBlock;
  int64_t* keys = c->alloc<int64_t>(m);
  int64_t* ref = c->alloc<int64_t>(m);
  int64_t* uid = c->alloc<int64_t>(m);
  if (!keys || !ref || !uid) return fail("ab_mesh_upload: device memory exhausted");
  k_win_keys<<<g256(m), 256, 0, c->st>>>(ne, nn, c->conn[k], c->n, keys, ref);
  thrust::stable_sort_by_key(thrust::cuda::par.on(c->st), keys, keys + m, ref);
  k_run_flags<<<g256(m), 256, 0, c->st>>>(m, keys, uid);
  thrust::inclusive_scan(thrust::cuda::par.on(c->st), uid, uid + m, uid);
  int64_t nwin = 0;
  cudaMemcpyAsync(&nwin, uid + m - 1, 8, cudaMemcpyDeviceToHost, c->st);
  cudaStreamSynchronize(c->st);
  int32_t* wnode = c->alloc<int32_t>(nwin);
  int32_t* wptr = c->alloc<int32_t>(nwin + 1);
  int64_t* wblk = c->alloc<int64_t>(nwin);
  uint16_t* wslot = c->alloc<uint16_t>(m);
  uint16_t* loc = c->alloc<uint16_t>(m);
  uint32_t* wref = c->alloc<uint32_t>(nblk * kWinBlock * nn);
  int64_t* blk_ptr = c->alloc<int64_t>(nblk + 1);
  int32_t* desc = c->alloc<int32_t>(4 * nblk);
  if (!wnode || !wptr || !wblk || !wslot || !loc || !wref || !blk_ptr || !desc)
    return fail("ab_mesh_upload: device memory exhausted");
  k_win_fill<<<g256(m), 256, 0, c->st>>>(m, nn, c->n, keys, ref, uid, wnode, wptr, wblk, wslot);
  const int32_t mi = (int32_t)m;
  cudaMemcpyAsync(wptr + nwin, &mi, 4, cudaMemcpyHostToDevice, c->st);
  thrust::lower_bound(thrust::cuda::par.on(c->st), wblk, wblk + nwin, thrust::counting_iterator<int64_t>(0),
                      thrust::counting_iterator<int64_t>(nblk + 1), blk_ptr);
  k_fill_u32<<<g256(nblk * kWinBlock * nn), 256, 0, c->st>>>(nblk * kWinBlock * nn, 0xFFFF0000u, wref);
  k_win_local<<<g256(m), 256, 0, c->st>>>(m, nn, ref, uid, blk_ptr, wslot, loc, wref);
  k_win_desc<<<g256(nblk), 256, 0, c->st>>>(nblk, blk_ptr, wptr, desc);
  // largest window
  std::vector<int64_t> bp(nblk + 1);
  cudaMemcpyAsync(bp.data(), blk_ptr, 8 * (nblk + 1), cudaMemcpyDeviceToHost, c->st);
  cudaStreamSynchronize(c->st);
  int64_t wmax = 1;
  for (int64_t b = 0; b < nblk; ++b) wmax = bp[b + 1] - bp[b] > wmax ? bp[b + 1] - bp[b] : wmax;
  AB_TRY(check_launch("ab_mesh_upload: windows"));
  AB_TRY(ab_set_windows(c->conn[k], kWinBlock, blk_ptr, wnode, wptr, wslot, loc, desc, (int32_t)wmax));
  return ab_set_window_refs(c->conn[k], wref);
}

// Unique (row, col) pairs of all element node pairs: CSR pattern (row-major).
int csr_pattern(ab_ctx* c, int64_t chunk) {
  std::vector<int64_t*> parts;
  std::vector<int64_t> sizes;
  for (int k = 0; k < c->mesh.n_cat; ++k) {
    const int nn = kNodeNN[c->mesh.cat[k].rule];
    const int64_t ne = c->mesh.cat[k].n_elem;
    for (int64_t e0 = 0; e0 < ne; e0 += chunk) {
      const int64_t e = ne - e0 < chunk ? ne - e0 : chunk;
      const int64_t m = e * nn * nn;
      int64_t* keys = nullptr;
      if (cudaMalloc(&keys, 8 * m) != cudaSuccess) return fail("ab_mesh_upload: device memory exhausted");
      k_pair_keys<<<g256(m), 256, 0, c->st>>>(e, nn, c->conn[k] + e0 * nn, c->n, keys);
      thrust::sort(thrust::cuda::par.on(c->st), keys, keys + m);
      int64_t* end = thrust::unique(thrust::cuda::par.on(c->st), keys, keys + m);
      parts.push_back(keys);
      sizes.push_back(end - keys);
    }
  }
  int64_t total = 0;
  for (int64_t s : sizes) total += s;
  int64_t* all = nullptr;
  if (cudaMalloc(&all, 8 * (total > 0 ? total : 1)) != cudaSuccess) return fail("ab_mesh_upload: device memory exhausted");
  int64_t off = 0;
  for (size_t i = 0; i < parts.size(); ++i) {
    cudaMemcpyAsync(all + off, parts[i], 8 * sizes[i], cudaMemcpyDeviceToDevice, c->st);
    off += sizes[i];
  }
  cudaStreamSynchronize(c->st);
  for (int64_t* q : parts) cudaFree(q);
  thrust::sort(thrust::cuda::par.on(c->st), all, all + total);
  const int64_t nnz = thrust::unique(thrust::cuda::par.on(c->st), all, all + total) - all;
  c->nnz = nnz;
  c->rp = c->alloc<int64_t>(c->n + 1);
  c->cols = c->alloc<int32_t>(nnz);
  if (!c->rp || !c->cols) { cudaFree(all); return fail("ab_mesh_upload: device memory exhausted"); }
  k_split_keys<<<g256(nnz), 256, 0, c->st>>>(nnz, all, c->n, nullptr, c->cols);
  // row_ptr[i] = first key >= i * n
  thrust::lower_bound(thrust::cuda::par.on(c->st), all, all + nnz,
                      thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), RowStart{c->n}),
                      thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(c->n + 1), RowStart{c->n}),
                      c->rp);
  cudaStreamSynchronize(c->st);
  cudaFree(all);
  return check_launch("ab_mesh_upload: csr pattern");
}

}  // namespace

extern "C" {

int ab_ctx_create(int32_t device, ab_ctx** out) {
  if (!out) return fail("ab_ctx_create: null output");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail("ab_ctx_create: no such CUDA device");
  if (cudaSetDevice(device) != cudaSuccess) return fail("ab_ctx_create: cudaSetDevice failed");
  ab_ctx* c = new ab_ctx();
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail("ab_ctx_create: cannot create the setup stream");
  }
  *out = c;
  return AB_OK;
}

int ab_ctx_destroy(ab_ctx* c) {
  if (!c) return AB_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  cudaStream_t s = c->st;
  delete c;
  cudaStreamDestroy(s);
  return AB_OK;
}

int ab_mesh_upload(ab_ctx* c, const ab_mesh_desc* d) {
  if (!c || !d) return fail("ab_mesh_upload: null argument");
  if (c->ready) return fail("ab_mesh_upload: the context already holds a mesh");
  if (d->n_nodes <= 0 || !d->coords) return fail("ab_mesh_upload: no nodes");
  if (d->n_cat < 1 || d->n_cat > 5) return fail("ab_mesh_upload: 1..5 categories");
  cudaSetDevice(c->device);
  const int64_t n = d->n_nodes;
  c->n = n;
  c->phys = d->phys;
  // nodes: f64 [n][4]
  double* c3 = c->alloc<double>(3 * n);
  AB_ALLOC(c->coords4, double, 4 * n);
  if (!c3) return fail("ab_mesh_upload: device memory exhausted");
  cudaMemcpyAsync(c3, d->coords, 24 * n, cudaMemcpyDefault, c->st);
  k_expand34<<<g256(n), 256, 0, c->st>>>(n, c3, c->coords4);
  c->mesh.n_nodes = n;
  c->mesh.coords = c->coords4;
  for (int a = 0; a < 3; ++a) c->mesh.period[a] = d->period[a];
  c->mesh.n_cat = d->n_cat;
  // categories: upload, then SFC order of the elements (Hilbert key of the
  // centroid in the box of all centroids, stable: device.py reorder_sfc)
  std::vector<double*> cents(d->n_cat);
  for (int k = 0; k < d->n_cat; ++k) {
    const int rule = d->cat[k].rule;
    if (rule < 0 || rule > 4) return fail("ab_mesh_upload: unknown rule");
    const int nn = kNodeNN[rule];
    const int64_t ne = d->cat[k].n_elem;
    if (ne < 0 || (ne > 0 && !d->cat[k].conn)) return fail("ab_mesh_upload: bad category");
    int32_t* raw = c->alloc<int32_t>(ne * nn);
    if (!raw) return fail("ab_mesh_upload: device memory exhausted");
    cudaMemcpyAsync(raw, d->cat[k].conn, 4 * ne * nn, cudaMemcpyDefault, c->st);
    c->mesh.cat[k] = ab_category{rule, 0, ne, raw};
    cents[k] = c->alloc<double>(3 * ne);
    if (!cents[k]) return fail("ab_mesh_upload: device memory exhausted");
    if (ne) AB_TRY(ab_centroids(&c->mesh, k, cents[k], c->st));
  }
  MinMax3 mm;
  for (int a = 0; a < 3; ++a) { mm.lo[a] = 1e308; mm.hi[a] = -1e308; }
  for (int k = 0; k < d->n_cat; ++k)
    if (c->mesh.cat[k].n_elem) mm = MMJoin{}(mm, minmax(c, cents[k], c->mesh.cat[k].n_elem, 3));
  for (int k = 0; k < d->n_cat; ++k) {
    const int nn = kNodeNN[c->mesh.cat[k].rule];
    const int64_t ne = c->mesh.cat[k].n_elem;
    int64_t* order = c->alloc<int64_t>(ne);
    AB_ALLOC(c->conn[k], int32_t, ne * nn);
    if (!order) return fail("ab_mesh_upload: device memory exhausted");
    if (ne) {
      AB_TRY(hilbert_order(c, ne, cents[k], mm, order));
      k_gather_rows<<<g256(ne * nn), 256, 0, c->st>>>(ne, nn, c->mesh.cat[k].conn, order, c->conn[k]);
    }
    c->mesh.cat[k].conn = c->conn[k];
  }
  // node windows (pipelined element kernels) + Vreman filter width
  for (int k = 0; k < d->n_cat; ++k) {
    const int64_t ne = c->mesh.cat[k].n_elem;
    if (!ne) continue;
    AB_TRY(build_windows(c, k, ne, kNodeNN[c->mesh.cat[k].rule]));
    AB_ALLOC(c->delta2[k], double, ne);
    AB_TRY(ab_filter_width(&c->mesh, k, c->delta2[k], c->st));
    AB_TRY(ab_set_filter_width(c->conn[k], ne, c->delta2[k]));
  }
  // lumped mass (K1) and its inverse
  AB_ALLOC(c->ml, double, n);
  AB_ALLOC(c->minv, double, n);
  for (int k = 0; k < d->n_cat; ++k)
    if (c->mesh.cat[k].n_elem) AB_TRY(ab_mass(&c->mesh, k, nullptr, nullptr, c->ml, 128, c->st));
  AB_TRY(ab_reciprocal(n, c->ml, c->minv, c->st));
  // Laplacian with Dirichlet rows/cols -> identity; gradient operator on its pattern
  AB_TRY(csr_pattern(c, (int64_t)1 << 22));
  double* lv = c->alloc<double>(c->nnz);
  double* gv[3] = {c->alloc<double>(c->nnz), c->alloc<double>(c->nnz), c->alloc<double>(c->nnz)};
  uint8_t* fixed = c->alloc<uint8_t>(n);
  if (!lv || !gv[0] || !gv[1] || !gv[2] || !fixed) return fail("ab_mesh_upload: device memory exhausted");
  AB_TRY(ab_laplacian_csr(&c->mesh, c->rp, c->cols, lv, c->st));
  bool any_fixed = false;
  if (d->p_fixed) {
    cudaMemcpyAsync(fixed, d->p_fixed, n, cudaMemcpyDefault, c->st);
    for (int64_t i = 0; i < n && !any_fixed; ++i) any_fixed = d->p_fixed[i] != 0;
    if (any_fixed) AB_TRY(ab_csr_dirichlet(n, c->rp, c->cols, lv, fixed, c->st));
  }
  AB_TRY(ab_gradop_csr(&c->mesh, c->rp, c->cols, gv[0], gv[1], gv[2], c->st));
  {
    int64_t* sp = nullptr;
    int32_t* scol = nullptr;
    double* sv[3];
    AB_TRY(to_sell(c, n, c->rp, c->cols, gv[0], &sp, &scol, &sv[0], nullptr, nullptr));
    for (int a = 1; a < 3; ++a) {
      int64_t* sp2 = nullptr;
      int32_t* scol2 = scol;  // same pattern: the columns are rewritten identically
      AB_TRY(to_sell(c, n, c->rp, c->cols, gv[a], &sp2, &scol2, &sv[a], nullptr, nullptr));
    }
    c->B3 = ab_sell3{n, (n + 31) / 32, sp, scol, sv[0], sv[1], sv[2]};
  }
  // pressure system in the Hilbert order of the nodes: P L P^T (solver.py permute_matrix)
  {
    double* diag = c->alloc<double>(n);
    double* c3n = c->alloc<double>(3 * n);
    int64_t* iperm = c->alloc<int64_t>(n);
    AB_ALLOC(c->perm, int64_t, n);
    if (!diag || !c3n || !iperm) return fail("ab_mesh_upload: device memory exhausted");
    k_coords3<<<g256(n), 256, 0, c->st>>>(n, c->coords4, c3n);
    AB_TRY(hilbert_order(c, n, c3n, minmax(c, c3n, n, 3), c->perm));
    k_invert<<<g256(n), 256, 0, c->st>>>(n, c->perm, iperm);
    int64_t* row = c->alloc<int64_t>(c->nnz);
    int64_t* keys = c->alloc<int64_t>(c->nnz);
    int64_t* idx = c->alloc<int64_t>(c->nnz);
    int64_t* rp2 = c->alloc<int64_t>(n + 1);
    int32_t* cols2 = c->alloc<int32_t>(c->nnz);
    double* v2 = c->alloc<double>(c->nnz);
    if (!row || !keys || !idx || !rp2 || !cols2 || !v2) return fail("ab_mesh_upload: device memory exhausted");
    k_row_of<<<g256(n), 256, 0, c->st>>>(n, c->rp, row);
    k_perm_keys<<<g256(c->nnz), 256, 0, c->st>>>(c->nnz, row, c->cols, iperm, n, keys, idx);
    thrust::sort_by_key(thrust::cuda::par.on(c->st), keys, keys + c->nnz, idx);
    k_split_keys<<<g256(c->nnz), 256, 0, c->st>>>(c->nnz, keys, n, row, cols2);
    k_gather_f64<<<g256(c->nnz), 256, 0, c->st>>>(c->nnz, lv, idx, v2);
    thrust::lower_bound(thrust::cuda::par.on(c->st), row, row + c->nnz, thrust::counting_iterator<int64_t>(0),
                        thrust::counting_iterator<int64_t>(n + 1), rp2);
    int64_t* sp = nullptr;
    int32_t* scol = nullptr;
    double* sv = nullptr;
    int64_t stored = 0;
    AB_TRY(to_sell(c, n, rp2, cols2, v2, &sp, &scol, &sv, diag, &stored));
    int64_t maxw = 0;
    {
      std::vector<int64_t> h((n + 31) / 32 + 1);
      cudaMemcpyAsync(h.data(), sp, 8 * h.size(), cudaMemcpyDeviceToHost, c->st);
      cudaStreamSynchronize(c->st);
      for (size_t s = 0; s + 1 < h.size(); ++s) maxw = (h[s + 1] - h[s]) / 32 > maxw ? (h[s + 1] - h[s]) / 32 : maxw;
    }
    c->Lp = ab_sell{n, (n + 31) / 32, maxw, sp, scol, sv};
    AB_ALLOC(c->dinv_p, double, n);
    AB_ALLOC(c->fixed_p, uint8_t, n);
    k_gather_u8<<<g256(n), 256, 0, c->st>>>(n, fixed, c->perm, c->fixed_p);
    if (any_fixed) k_set_diag_fixed<<<g256(n), 256, 0, c->st>>>(n, c->fixed_p, diag);
    AB_TRY(ab_reciprocal(n, diag, c->dinv_p, c->st));
    AB_TRY(build_tiled_cg(c, n, rp2, cols2, v2, iperm));
  }
  // CG workspace (two-kernel form: grouped grid reductions)
  const int64_t nb = (n + 255) / 256 + 1;
  const int64_t ng = (nb + 63) / 64 + 1;
  AB_ALLOC(c->x, double, n);
  AB_ALLOC(c->r, double, n);
  AB_ALLOC(c->z, double, n);
  AB_ALLOC(c->p, double, n);
  AB_ALLOC(c->q, double, n);
  AB_ALLOC(c->xn, double, n);
  AB_ALLOC(c->red, double, 8);
  AB_ALLOC(c->sc, double, 8);
  AB_ALLOC(c->part, double, 5 * (nb + ng) + 8);
  AB_ALLOC(c->cnt, uint32_t, ng + 2);
  // state
  AB_ALLOC(c->U0, double, 4 * n);
  AB_ALLOC(c->U, double, 4 * n);
  AB_ALLOC(c->R, double, 4 * n);
  AB_ALLOC(c->GP, double, 4 * n);
  AB_ALLOC(c->P, double, n);
  AB_ALLOC(c->Bv, double, n);
  AB_ALLOC(c->stage, double, 3 * n);
  // velocity Dirichlet list
  if (d->u_fixed) {
    std::vector<int32_t> idx;
    std::vector<uint8_t> mk;
    std::vector<double> vals;
    for (int64_t i = 0; i < n; ++i)
      if (d->u_fixed[i] & 7) {
        idx.push_back((int32_t)i);
        mk.push_back(d->u_fixed[i] & 7);
        for (int a = 0; a < 3; ++a) vals.push_back(d->u_values ? d->u_values[3 * i + a] : 0.0);
      }
    c->nbc = (int64_t)idx.size();
    if (c->nbc) {
      AB_ALLOC(c->bc_idx, int32_t, c->nbc);
      AB_ALLOC(c->bc_mask, uint8_t, c->nbc);
      AB_ALLOC(c->bc_vals, double, 3 * c->nbc);
      cudaMemcpyAsync(c->bc_idx, idx.data(), 4 * c->nbc, cudaMemcpyHostToDevice, c->st);
      cudaMemcpyAsync(c->bc_mask, mk.data(), c->nbc, cudaMemcpyHostToDevice, c->st);
      cudaMemcpyAsync(c->bc_vals, vals.data(), 24 * c->nbc, cudaMemcpyHostToDevice, c->st);
      cudaStreamSynchronize(c->st);  // host vectors go out of scope
    }
  }
  // wall-model faces (boundary assembly, Algorithm 1 line 4)
  if (d->n_wall_faces > 0) {
    int32_t *f = nullptr, *o = nullptr;
    AB_ALLOC(f, int32_t, 4 * d->n_wall_faces);
    AB_ALLOC(o, int32_t, 4 * d->n_wall_faces);
    cudaMemcpyAsync(f, d->wall_face, 16 * d->n_wall_faces, cudaMemcpyDefault, c->st);
    cudaMemcpyAsync(o, d->wall_off, 16 * d->n_wall_faces, cudaMemcpyDefault, c->st);
    c->wall = ab_wall{d->n_wall_faces, f, o, 0, nullptr, nullptr, nullptr, nullptr};
  }
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return check_launch("ab_mesh_upload");
  c->ready = true;
  return check_launch("ab_mesh_upload");
}

int ab_ctx_info(const ab_ctx* c, ab_ctx_info_t* info) {
  if (!c || !info) return fail("ab_ctx_info: null argument");
  memset(info, 0, sizeof(*info));
  info->n_nodes = c->n;
  info->nnz = c->nnz;
  info->n_cat = c->mesh.n_cat;
  for (int k = 0; k < c->mesh.n_cat; ++k) info->n_elem[k] = c->mesh.cat[k].n_elem;
  info->n_velocity_bc = c->nbc;
  info->n_wall_faces = c->wall.n_faces;
  info->ready = c->ready ? 1 : 0;
  return AB_OK;
}

static int apply_bc(ab_ctx* c, double* u4, cudaStream_t s) {
  if (!c->nbc) return AB_OK;
  return ab_apply_velocity_bc(c->nbc, c->bc_idx, c->bc_mask, c->bc_vals, u4, s);
}

int ab_state_set(ab_ctx* c, const double* u, const double* p, void* stream) {
  if (!c || !c->ready) return fail("ab_state_set: no mesh uploaded");
  if (!u || !p) return fail("ab_state_set: null state");
  cudaStream_t s = S(stream);
  const int64_t n = c->n;
  if (cudaMemcpyAsync(c->stage, u, 24 * n, cudaMemcpyDefault, s) != cudaSuccess ||
      cudaMemcpyAsync(c->P, p, 8 * n, cudaMemcpyDefault, s) != cudaSuccess)
    return fail("ab_state_set: copy failed");
  k_expand34<<<g256(n), 256, 0, s>>>(n, c->stage, c->U0);
  AB_TRY(apply_bc(c, c->U0, s));
  cudaMemsetAsync(c->GP, 0, 32 * n, s);
  AB_TRY(ab_gradop_grad(&c->B3, c->P, 1.0, c->GP, s));  // G p^n
  return check_launch("ab_state_set");
}

int ab_state_get(ab_ctx* c, double* u, double* p, void* stream) {
  if (!c || !c->ready) return fail("ab_state_get: no mesh uploaded");
  cudaStream_t s = S(stream);
  const int64_t n = c->n;
  if (u) {
    k_compact43<<<g256(n), 256, 0, s>>>(n, c->U0, c->stage);
    if (cudaMemcpyAsync(u, c->stage, 24 * n, cudaMemcpyDefault, s) != cudaSuccess) return fail("ab_state_get: copy failed");
  }
  if (p && cudaMemcpyAsync(p, c->P, 8 * n, cudaMemcpyDefault, s) != cudaSuccess) return fail("ab_state_get: copy failed");
  return check_launch("ab_state_get");
}

int ab_step(ab_ctx* c, double dt, int32_t cg_iters, void* stream) {
  if (!c || !c->ready) return fail("ab_step: no mesh uploaded");
  if (!(dt > 0.0) || cg_iters < 0) return fail("ab_step: dt must be > 0 and cg_iters >= 0");
  cudaStream_t s = S(stream);
  const int64_t n = c->n;
  static const double A[3] = {0.0, 0.75, 1.0 / 3.0}, B[3] = {1.0, 0.25, 2.0 / 3.0};  // SSP-RK3 (timestep.py)
  const double k = dt / c->phys.rho;
  for (int stg = 0; stg < 3; ++stg) {
    const double* uin = stg == 0 ? c->U0 : c->U;
    AB_TRY(ab_momentum_rhs(&c->mesh, &c->phys, uin, c->R, s));                        // K2
    if (c->wall.n_faces) AB_TRY(ab_wall_traction(&c->wall, &c->phys, c->coords4, uin, c->R, s));  // K8
    AB_TRY(ab_rk_stage(n, A[stg], B[stg], k, c->U0, uin, c->R, c->GP, c->minv, c->U, s));         // K3
    AB_TRY(apply_bc(c, c->U, s));
  }
  AB_TRY(ab_gradop_div(&c->B3, c->U, -c->phys.rho / dt, c->Bv, s));  // K4: b = -(rho/dt) D u_3
  if (c->tiled) {
    // K5: tiled single-pass CG on S P L P^T S (= Jacobi-PCG), one kernel per iteration
    AB_TRY(ab_cg_tile_init(n, c->perm, c->Bv, 1, c->fixed_p, c->s_p, nullptr, c->xp, c->rq[0], c->red, c->sc,
                           c->part, c->cnt, s));
    for (int it = 0; it < cg_iters; ++it)
      AB_TRY(ab_cg_tile_iter(&c->Lu, &c->tmap, c->rq[it & 1], c->rq[(it + 1) & 1], c->xp, nullptr, c->red, c->part,
                             c->cnt, s));
    AB_TRY(ab_cg_tile_finish(n, c->iperm, c->s_p, c->xp, c->red, cg_iters > 0 ? 1 : 0, c->xn, s));
  } else {
    // K5: Jacobi-PCG on P L P^T (b gathered in, x scattered out)
    AB_TRY(ab_cg_init_perm(n, c->perm, c->Bv, 1, c->fixed_p, c->dinv_p, c->x, c->r, c->z, c->p, c->q, c->red, c->sc,
                           c->part, c->cnt, s));
    for (int it = 0; it < cg_iters; ++it) {
      AB_TRY(ab_cg_spmv(&c->Lp, c->z, c->p, c->q, nullptr, 1, nullptr, c->red, c->sc, c->part, c->cnt, s));
      AB_TRY(ab_cg_update(n, c->p, c->q, c->dinv_p, c->x, c->r, c->z, nullptr, c->red, c->sc, c->part, c->cnt, s));
    }
    AB_TRY(ab_perm_scatter(n, c->perm, c->x, c->xn, s));
  }
  // K6 + K7: u = u_3 - dt/rho M^-1 B dp; p += dp; Gp += B dp
  AB_TRY(ab_gradop_correct(&c->B3, c->xn, k, c->U, c->U0, c->minv, c->P, c->GP, s));
  AB_TRY(apply_bc(c, c->U0, s));
  return check_launch("ab_step");
}

}  // extern "C"
