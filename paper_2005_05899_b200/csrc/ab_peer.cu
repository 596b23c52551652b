// Peer-memory interface exchange and the decomposed CG for subdomains too
// large to stay on chip (include/alyab200.h).
//
// Every rank owns the buffers its neighbours write into (receive slots,
// arrival counters, reduction records); the neighbours reach them through
// CUDA IPC mappings (NVLink / NVSwitch peer stores) or, for ranks sharing one
// GPU in one process, as plain device pointers.  Progress state lives in
// device memory, so no launch argument changes between steps and the whole
// multi-rank step is graph-capturable.  The interface sums add the sharers'
// partials in ascending global rank order (this rank's own partial at its
// position), so duplicated interface values stay bitwise identical across
// ranks.
#include "ab_cg_common.cuh"

namespace ab {

static_assert(sizeof(ab_peer_halo) == 272, "ab_peer_halo layout (mirrored by _lib.AbPeerHalo)");
static_assert(sizeof(ab_ddcg2_rank) == 568, "ab_ddcg2_rank layout (mirrored by _lib.AbDdcg2Rank)");

constexpr int kPeerBlock = 256;
constexpr long long kPeerTimeoutNs = 10000000000ll;

__device__ __forceinline__ long long peer_time() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acq_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rel_f64(double* p, double v) {
  asm volatile("st.release.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_rlx_f64(double* p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_acq_f64(const double* p) {
  double v;
  asm volatile("ld.acquire.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_rlx_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
// Interface sum of an element-assembled nodal field
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kPeerBlock) k_halo_put(ab_peer_halo h, const double* __restrict__ f, int ncomp,
                                                         int stride) {
  const unsigned long long ev = h.state[AB_PS_EV];
  const size_t par = (size_t)(ev & 1ull);
  const size_t M = (size_t)h.max_shared;
  for (int i = blockIdx.x * kPeerBlock + threadIdx.x; i < h.n_if; i += gridDim.x * kPeerBlock) {
    const int64_t node = h.if_node[i];
    double v[3];
    for (int c = 0; c < ncomp; ++c) v[c] = f[node * stride + c];
    for (int e = h.if_ptr[i]; e < h.if_ptr[i + 1]; ++e) {
      const int q = h.if_rank[e];
      int k = 0;
      while (h.nbr_rank[k] != q) ++k;
      double* dst = h.nbr_recv[k] + ((par * h.n_ranks + h.rank) * M + (size_t)h.if_slot[e]) * 3;
      for (int c = 0; c < ncomp; ++c) dst[c] = v[c];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int k = 0; k < h.n_nbr; ++k) red_rel_u64(h.nbr_cnt[k], 1ull);
  }
}

__global__ void __launch_bounds__(kPeerBlock) k_halo_add(ab_peer_halo h, double* __restrict__ f, int ncomp,
                                                         int stride) {
  __shared__ int s_fail;
  const unsigned long long ev = h.state[AB_PS_EV];
  const size_t par = (size_t)(ev & 1ull);
  const size_t M = (size_t)h.max_shared;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  if ((int)threadIdx.x < h.n_nbr) {
    const int q = h.nbr_rank[threadIdx.x];
    const unsigned long long want = (ev + 1ull) * (unsigned long long)h.nbr_ncta[threadIdx.x];
    const long long t0 = peer_time();
    while (ld_acq_u64(h.cnt_in + q) < want) {
      if (peer_time() - t0 > kPeerTimeoutNs) { s_fail = 1; break; }
    }
  }
  __syncthreads();
  if (s_fail) {
    if (threadIdx.x == 0) h.state[AB_PS_FAIL] = 1ull;
  } else {
    for (int i = blockIdx.x * kPeerBlock + threadIdx.x; i < h.n_if; i += gridDim.x * kPeerBlock) {
      const int64_t node = h.if_node[i];
      double own[3], acc[3] = {0.0, 0.0, 0.0};
      for (int c = 0; c < ncomp; ++c) own[c] = f[node * stride + c];
      bool mine = false;
      for (int e = h.if_ptr[i]; e < h.if_ptr[i + 1]; ++e) {
        const int q = h.if_rank[e];
        if (!mine && q > h.rank) {
          for (int c = 0; c < ncomp; ++c) acc[c] += own[c];
          mine = true;
        }
        const double* src = h.recv + ((par * h.n_ranks + q) * M + (size_t)h.if_slot[e]) * 3;
        for (int c = 0; c < ncomp; ++c) acc[c] += __ldcg(src + c);
      }
      if (!mine)
        for (int c = 0; c < ncomp; ++c) acc[c] += own[c];
      for (int c = 0; c < ncomp; ++c) f[node * stride + c] = acc[c];
    }
  }
  // the last CTA to finish advances the exchange count (next parity)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long t = atomicAdd(h.state + AB_PS_TICK, 1ull);
    if (t + 1 == (ev + 1) * (unsigned long long)gridDim.x) {
      __threadfence();
      h.state[AB_PS_EV] = ev + 1;
    }
  }
}

// ---------------------------------------------------------------------------
// Decomposed CG, large subdomains
// ---------------------------------------------------------------------------
constexpr int kD2Block = 256;
constexpr int kD2IfGrid = 148;
constexpr int kRecStride = 10;  // doubles per (set, rank) record: up to 5 {value, epoch} pairs

// Grid-sum scratch: the row-parallel kernels (init, spmv, update, tile_iter:
// <= 5 values over <= ceil(n/64) + 1 blocks, tiles of >= 64 rows) use the
// front of `part` / `cnt`, the interface kernels the region behind it.
__host__ __device__ inline int64_t d2_front_blocks(int64_t n) { return (n + 63) / 64 + 1; }
__host__ __device__ inline int64_t d2_front_part(int64_t n) {
  const int64_t nb = d2_front_blocks(n);
  return 5 * (nb + (nb + kGroup - 1) / kGroup + 1) + 8;
}
__host__ __device__ inline int64_t d2_front_cnt(int64_t n) {
  return 2 + (d2_front_blocks(n) + kGroup - 1) / kGroup;
}

// Record of `set` published by rank `src`: NV values into every rank's
// record array (this rank's own included).
template <int NV>
__device__ __forceinline__ void d2_publish(const ab_ddcg2_rank& d, int set, const double (&v)[NV], double ep) {
  const int P = d.n_ranks;
  double* dst0 = d.rec + ((size_t)set * P + d.rank) * kRecStride;
#pragma unroll
  for (int k = 0; k < NV; ++k) st_rlx_f64(dst0 + 2 * k, v[k]);
  for (int q = 0; q < d.n_peers; ++q) {
    double* dst = d.peer_rec[q] + ((size_t)set * P + d.rank) * kRecStride;
#pragma unroll
    for (int k = 0; k < NV; ++k) st_rlx_f64(dst + 2 * k, v[k]);
  }
  // epochs after all values (release orders the value stores before them)
#pragma unroll
  for (int k = 0; k < NV; ++k) st_rel_f64(dst0 + 2 * k + 1, ep);
  for (int q = 0; q < d.n_peers; ++q) {
    double* dst = d.peer_rec[q] + ((size_t)set * P + d.rank) * kRecStride;
#pragma unroll
    for (int k = 0; k < NV; ++k) st_rel_f64(dst + 2 * k + 1, ep);
  }
}

// Every rank's record of `set` at epoch `ep`, summed in rank order; the same
// in every thread of the block.  Returns false on a timeout.
template <int NV>
__device__ __forceinline__ bool d2_collect(const ab_ddcg2_rank& d, int set, double ep, double (&out)[NV],
                                           double* sbuf /* [NV * P] shared */, int* sflag) {
  const int P = d.n_ranks;
  if ((int)threadIdx.x < P) {
    const double* rec = d.rec + ((size_t)set * P + threadIdx.x) * kRecStride;
    const long long t0 = peer_time();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double v = 0.0;
      for (;;) {
        if (ld_acq_f64(rec + 2 * k + 1) == ep) { v = ld_rlx_f64(rec + 2 * k); break; }
        if (peer_time() - t0 > kPeerTimeoutNs) { *sflag = 1; break; }
      }
      sbuf[k * P + threadIdx.x] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double acc = 0.0;
    for (int q = 0; q < P; ++q) acc += sbuf[k * P + q];
    out[k] = acc;
  }
  const bool ok = *sflag == 0;
  __syncthreads();
  return ok;
}

__global__ void __launch_bounds__(kD2Block) k_d2_init(ab_ddcg2_rank d, const double* __restrict__ b, double* b_zero,
                                                      double tol) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * kD2Block + threadIdx.x; i < d.n_rows;
       i += (int64_t)gridDim.x * kD2Block) {
    const int64_t ni = d.perm[i];
    double ri = b[ni];
    if (d.fixed && d.fixed[i]) ri = 0.0;
    const double w = d.own[i];
    if (d.scaled) {  // r' = D^-1/2 r; r.z = r'.r'; ||r||^2 = sum r'^2 / dinv when a tolerance is tested
      ri *= d.s[i];
      v[0] += w * ri * ri;
      v[1] += tol > 0.0 ? w * ri * ri / d.dinv[i] : w * ri * ri;
    } else {
      const double zi = d.dinv[i] * ri;
      d.z[i] = zi;
      v[0] += w * ri * zi;
      v[1] += w * ri * ri;
    }
    d.r[i] = ri;
    d.x[i] = 0.0;
    d.p[i] = 0.0;
    d.q[i] = 0.0;
  }
  double tot[2];
  if (grid_sum<2, kD2Block>(v, d.part, d.cnt, tot) && threadIdx.x == 0) {
    const double ep = d.scal[AB_D2_EPOCH] + 1.0;
    d.scal[AB_D2_EPOCH] = ep;
    d.scal[AB_D2_EPB] = ep;
    d.scal[AB_D2_IT] = 0.0;
    d.scal[AB_D2_DONE] = 0.0;
    d.scal[AB_D2_RZ0] = 0.0;
    d.scal[AB_D2_RZ0 + 1] = 0.0;
    d.scal[AB_D2_TOL] = tol;
    d2_publish<2>(d, 1, tot, ep);
  }
}

__global__ void k_d2_zero(int64_t n, double* b) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = 0.0;
}

__global__ void __launch_bounds__(kD2Block) k_d2_spmv(ab_ddcg2_rank d) {
  __shared__ double sbuf[2 * 32];
  __shared__ int sflag;
  if (d.scal[AB_D2_DONE] != 0.0) return;
  if (threadIdx.x == 0) sflag = 0;
  __syncthreads();
  const int it = (int)d.scal[AB_D2_IT];
  double t2[2];
  if (!d2_collect<2>(d, 1, d.scal[AB_D2_EPB], t2, sbuf, &sflag)) {
    if (threadIdx.x == 0) { d.scal[AB_D2_FAIL] = 1.0; d.scal[AB_D2_DONE] = 1.0; }
    return;
  }
  const double rz_new = t2[0], rr = t2[1];
  const double bb = it == 0 ? rr : d.scal[AB_D2_BB];
  const double tol = d.scal[AB_D2_TOL];
  if (tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) {  // identical decision in every block and rank
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      d.scal[AB_D2_DONE] = 1.0;
      d.scal[AB_D2_RR] = rr;
      if (it == 0) d.scal[AB_D2_BB] = bb;
    }
    return;
  }
  const double rz_old = d.scal[AB_D2_RZ0 + ((it + 1) & 1)];
  const double beta = it > 0 && rz_old != 0.0 ? rz_new / rz_old : 0.0;
  const int64_t i = (int64_t)blockIdx.x * kD2Block + threadIdx.x;
  double v[1] = {0.0};
  const double* zv = d.scaled ? d.r : d.z;  // the scaled form gathers r' where Jacobi gathers z
  if (i < d.n_rows) {
    const double az = sell_row_dot(d.slice_ptr, d.cols, d.vals, zv, i);
    if (i < d.n_if) {
      d.tif[i] = az;
      for (int e = d.send_ptr[i]; e < d.send_ptr[i + 1]; ++e) d.peer_recv[d.send_peer[e]][d.send_off[e]] = az;
    } else {
      const double pi = fma(beta, d.p[i], zv[i]);
      const double qi = fma(beta, d.q[i], az);
      d.p[i] = pi;
      d.q[i] = qi;
      v[0] = pi * qi;  // interior rows belong to this rank alone (own = 1)
    }
  }
  if ((int64_t)blockIdx.x * kD2Block < d.n_if) {  // a signalling block: its puts are complete
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int q = 0; q < d.n_peers; ++q)
        if (d.peer_nsig[q] > 0) red_rel_u64(d.peer_cnt[q], 1ull);
    }
  }
  double tot[1];
  if (grid_sum<1, kD2Block>(v, d.part, d.cnt, tot) && threadIdx.x == 0) {
    d.scal[AB_D2_PQI] = tot[0];
    d.scal[AB_D2_BETA] = beta;
    d.scal[AB_D2_RZ0 + (it & 1)] = rz_new;
    d.scal[AB_D2_RR] = rr;
    if (it == 0) d.scal[AB_D2_BB] = bb;
  }
}

// Tiled form of k_d2_spmv (d.tile_rows > 0): CTA b owns rows [b R, (b+1) R),
// stages z of its rows and ghost rows in shared memory and reads the slices
// with 16-bit tile-local columns (ab_cg_spmv_tile's scheme); the tiles
// holding interface rows come first and signal once their puts are done.
__global__ void __launch_bounds__(kD2Block) k_d2_spmv_tile(ab_ddcg2_rank d) {
  extern __shared__ __align__(16) double zs[];
  __shared__ double sbuf[2 * 32];
  __shared__ int sflag;
  if (d.scal[AB_D2_DONE] != 0.0) return;
  if (threadIdx.x == 0) sflag = 0;
  __syncthreads();
  const int it = (int)d.scal[AB_D2_IT];
  double t2[2];
  if (!d2_collect<2>(d, 1, d.scal[AB_D2_EPB], t2, sbuf, &sflag)) {
    if (threadIdx.x == 0) { d.scal[AB_D2_FAIL] = 1.0; d.scal[AB_D2_DONE] = 1.0; }
    return;
  }
  const double rz_new = t2[0], rr = t2[1];
  const double bb = it == 0 ? rr : d.scal[AB_D2_BB];
  const double tol = d.scal[AB_D2_TOL];
  if (tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) {  // identical decision in every block and rank
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      d.scal[AB_D2_DONE] = 1.0;
      d.scal[AB_D2_RR] = rr;
      if (it == 0) d.scal[AB_D2_BB] = bb;
    }
    return;
  }
  const double rz_old = d.scal[AB_D2_RZ0 + ((it + 1) & 1)];
  const double beta = it > 0 && rz_old != 0.0 ? rz_new / rz_old : 0.0;
  const double* zv = d.scaled ? d.r : d.z;  // the scaled form gathers r' where Jacobi gathers z
  const int R = d.tile_rows;
  const int64_t row0 = (int64_t)blockIdx.x * R;
  const int rows = (int)(d.n_rows - row0 < R ? d.n_rows - row0 : R);
  for (int k = threadIdx.x; k < rows; k += kD2Block) zs[k] = __ldcg(zv + row0 + k);
  const int g0 = d.tghost_ptr[blockIdx.x], ng = d.tghost_ptr[blockIdx.x + 1] - g0;
  for (int k = threadIdx.x; k < ng; k += kD2Block) zs[R + k] = __ldcg(zv + __ldg(d.tghost + g0 + k));
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nsl = (rows + 31) >> 5;
  double v[1] = {0.0};
  for (int sl = warp; sl < nsl; sl += kD2Block / 32) {
    const double az = sell_row_dot_smem<8>(d.slice_ptr + (row0 >> 5), d.tcols, d.vals, zs, sl, lane);
    const int li = sl * 32 + lane;
    if (li < rows) {
      const int64_t i = row0 + li;
      if (i < d.n_if) {
        d.tif[i] = az;
        for (int e = d.send_ptr[i]; e < d.send_ptr[i + 1]; ++e) d.peer_recv[d.send_peer[e]][d.send_off[e]] = az;
      } else {
        const double pi = fma(beta, d.p[i], zs[li]);
        const double qi = fma(beta, d.q[i], az);
        d.p[i] = pi;
        d.q[i] = qi;
        v[0] += pi * qi;  // interior rows belong to this rank alone (own = 1)
      }
    }
  }
  if (row0 < d.n_if) {  // a signalling tile: its puts are complete
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int q = 0; q < d.n_peers; ++q)
        if (d.peer_nsig[q] > 0) red_rel_u64(d.peer_cnt[q], 1ull);
    }
  }
  double tot[1];
  if (grid_sum<1, kD2Block>(v, d.part, d.cnt, tot) && threadIdx.x == 0) {
    d.scal[AB_D2_PQI] = tot[0];
    d.scal[AB_D2_BETA] = beta;
    d.scal[AB_D2_RZ0 + (it & 1)] = rz_new;
    d.scal[AB_D2_RR] = rr;
    if (it == 0) d.scal[AB_D2_BB] = bb;
  }
}

__global__ void __launch_bounds__(kD2Block) k_d2_iface(ab_ddcg2_rank d) {
  __shared__ int sflag;
  if (d.scal[AB_D2_DONE] != 0.0) return;
  if (threadIdx.x == 0) sflag = 0;
  __syncthreads();
  const double hev = d.scal[AB_D2_HEV];
  if ((int)threadIdx.x < d.n_peers && d.peer_nsig[threadIdx.x] > 0) {
    const int q = d.peer_rank[threadIdx.x];
    const unsigned long long want = (unsigned long long)(hev + 1.0) * (unsigned long long)d.peer_nsig[threadIdx.x];
    const long long t0 = peer_time();
    while (ld_acq_u64(d.cnt_in + q) < want) {
      if (peer_time() - t0 > kPeerTimeoutNs) { sflag = 1; break; }
    }
  }
  __syncthreads();
  const bool failed = sflag != 0;
  const double beta = d.scal[AB_D2_BETA];
  double v[1] = {0.0};
  if (!failed) {
    for (int64_t i = (int64_t)blockIdx.x * kD2Block + threadIdx.x; i < d.n_if; i += (int64_t)gridDim.x * kD2Block) {
      const double own_t = d.tif[i];
      double t = 0.0;
      bool mine = false;
      for (int e = d.recv_ptr[i]; e < d.recv_ptr[i + 1]; ++e) {
        if (!mine && d.recv_rank[e] > d.rank) { t += own_t; mine = true; }
        t += __ldcg(d.recv + d.recv_off[e]);
      }
      if (!mine) t += own_t;
      const double pi = fma(beta, d.p[i], d.scaled ? d.r[i] : d.z[i]);
      const double qi = fma(beta, d.q[i], t);
      d.p[i] = pi;
      d.q[i] = qi;
      v[0] += d.own[i] * pi * qi;
    }
  }
  double tot[1];
  // (part/cnt behind the SpMV's: ab_ddcg2_part_size)
  double* part = d.part + d2_front_part(d.n_rows);
  uint32_t* cnt = d.cnt + d2_front_cnt(d.n_rows);
  if (grid_sum<1, kD2Block>(v, part, cnt, tot) && threadIdx.x == 0) {
    d.scal[AB_D2_HEV] = hev + 1.0;
    if (failed) {
      d.scal[AB_D2_FAIL] = 1.0;
      d.scal[AB_D2_DONE] = 1.0;
      return;
    }
    const double ep = d.scal[AB_D2_EPOCH] + 1.0;
    d.scal[AB_D2_EPOCH] = ep;
    d.scal[AB_D2_EPA] = ep;
    const double pq[1] = {d.scal[AB_D2_PQI] + tot[0]};
    d2_publish<1>(d, 0, pq, ep);
  }
}

__global__ void __launch_bounds__(kD2Block) k_d2_update(ab_ddcg2_rank d) {
  __shared__ double sbuf[32];
  __shared__ int sflag;
  if (d.scal[AB_D2_DONE] != 0.0) return;
  if (threadIdx.x == 0) sflag = 0;
  __syncthreads();
  double t1[1];
  if (!d2_collect<1>(d, 0, d.scal[AB_D2_EPA], t1, sbuf, &sflag)) {
    if (threadIdx.x == 0) { d.scal[AB_D2_FAIL] = 1.0; d.scal[AB_D2_DONE] = 1.0; }
    return;
  }
  const int it = (int)d.scal[AB_D2_IT];
  const double rz = d.scal[AB_D2_RZ0 + (it & 1)];
  const double alpha = t1[0] != 0.0 ? rz / t1[0] : 0.0;
  double v[2] = {0.0, 0.0};
  const bool true_norm = d.scal[AB_D2_TOL] > 0.0;
  const int64_t n = d.n_rows;
  // two rows per thread with 16-byte accesses, grid-stride (fewer blocks,
  // so fewer record collections); interior rows have weight 1
  for (int64_t k = (int64_t)blockIdx.x * kD2Block + threadIdx.x; 2 * k < n; k += (int64_t)gridDim.x * kD2Block) {
    const int64_t i = 2 * k;
    double rr2[2], w[2];
    if (i + 1 < n) {
      const double2 pv = *reinterpret_cast<const double2*>(d.p + i);
      const double2 qv = *reinterpret_cast<const double2*>(d.q + i);
      const double2 xv = *reinterpret_cast<const double2*>(d.x + i);
      const double2 rv = *reinterpret_cast<const double2*>(d.r + i);
      *reinterpret_cast<double2*>(d.x + i) = make_double2(fma(alpha, pv.x, xv.x), fma(alpha, pv.y, xv.y));
      rr2[0] = fma(-alpha, qv.x, rv.x);
      rr2[1] = fma(-alpha, qv.y, rv.y);
      *reinterpret_cast<double2*>(d.r + i) = make_double2(rr2[0], rr2[1]);
    } else {
      d.x[i] = fma(alpha, d.p[i], d.x[i]);
      rr2[0] = fma(-alpha, d.q[i], d.r[i]);
      d.r[i] = rr2[0];
      rr2[1] = 0.0;
    }
    w[0] = i < d.n_if ? d.own[i] : 1.0;
    w[1] = i + 1 < n ? (i + 1 < d.n_if ? d.own[i + 1] : 1.0) : 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && i + 1 >= n) break;
      const double rk = rr2[h];
      if (d.scaled) {
        v[0] += w[h] * rk * rk;
        v[1] += true_norm ? w[h] * rk * rk / d.dinv[i + h] : w[h] * rk * rk;
      } else {
        const double zk = d.dinv[i + h] * rk;
        d.z[i + h] = zk;
        v[0] += w[h] * rk * zk;
        v[1] += w[h] * rk * rk;
      }
    }
  }
  double tot[2];
  if (grid_sum<2, kD2Block>(v, d.part, d.cnt, tot) && threadIdx.x == 0) {
    const double ep = d.scal[AB_D2_EPOCH] + 1.0;
    d.scal[AB_D2_EPOCH] = ep;
    d.scal[AB_D2_EPB] = ep;
    d.scal[AB_D2_IT] = (double)(it + 1);
    d2_publish<2>(d, 1, tot, ep);
  }
}

// ---------------------------------------------------------------------------
// Single-pass decomposed CG (d.single_pass, scaled form, tiled): TWO launches
// per iteration instead of three.  k_d2_tile_iter forms r'_j = r'_{j-1} -
// alpha q_{j-1} while staging the tile and its ghost rows (16-byte (r', q)
// pairs, ping-pong), x_j, p_j for every row, q_j and the dots for the
// interior rows, and the interface rows' partial products -> peers (their
// q_{j-1} parked in the output pair); k_d2_tile_iface sums the interface
// partials in rank order into q_j, adds the interface rows' weighted dots and
// publishes {r'r', ||r||^2 form, p.q, r'.q, q.q} (record sets alternate
// between iterations, so a set is rewritten only after every rank collected
// it).  beta_{j-1} comes from the recurrence r'r'_j = r'r'_{j-1} - 2 alpha
// r'.q_{j-1} + alpha^2 q.q_{j-1} (the single-domain ab_cg_tile_iter's
// scheme); the finish adds the last alpha p unless the solve converged.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kD2Block) k_d2_init_sp(ab_ddcg2_rank d, const double* __restrict__ b, double tol) {
  double v[2] = {0.0, 0.0};
  double2* rq = reinterpret_cast<double2*>(d.rq[0]);
  double2* xp = reinterpret_cast<double2*>(d.xp);
  for (int64_t i = (int64_t)blockIdx.x * kD2Block + threadIdx.x; i < d.n_rows;
       i += (int64_t)gridDim.x * kD2Block) {
    double ri = b[d.perm[i]];
    if (d.fixed && d.fixed[i]) ri = 0.0;
    ri *= d.s[i];
    const double w = i < d.n_if ? d.own[i] : 1.0;
    v[0] += w * ri * ri;
    v[1] += tol > 0.0 ? w * ri * ri / d.dinv[i] : w * ri * ri;
    rq[i] = make_double2(ri, 0.0);
    xp[i] = make_double2(0.0, 0.0);
  }
  double tot[2];
  if (grid_sum<2, kD2Block>(v, d.part, d.cnt, tot) && threadIdx.x == 0) {
    const double ep = d.scal[AB_D2_EPOCH] + 1.0;
    d.scal[AB_D2_EPOCH] = ep;
    d.scal[AB_D2_EPB] = ep;
    d.scal[AB_D2_IT] = 0.0;
    d.scal[AB_D2_DONE] = 0.0;
    d.scal[AB_D2_TOL] = tol;
    const double rec[5] = {tot[0], tot[1], 0.0, 0.0, 0.0};  // alpha_{-1} = 0: the first iteration keeps x = 0
    d2_publish<5>(d, 0, rec, ep);
  }
}

__global__ void __launch_bounds__(kD2Block) k_d2_tile_iter(ab_ddcg2_rank d) {
  extern __shared__ __align__(16) double qs[];  // [R] q_{j-1} of the tile's rows, then zs
  __shared__ double sbuf[5 * 32];
  __shared__ int sflag;
  if (d.scal[AB_D2_DONE] != 0.0) return;
  if (threadIdx.x == 0) sflag = 0;
  __syncthreads();
  const int it = (int)d.scal[AB_D2_IT];
  double t[5];
  if (!d2_collect<5>(d, it & 1, d.scal[AB_D2_EPB], t, sbuf, &sflag)) {
    if (threadIdx.x == 0) { d.scal[AB_D2_FAIL] = 1.0; d.scal[AB_D2_DONE] = 1.0; }
    return;
  }
  const double RR = t[0], rr = t[1], PQ = t[2], RQ = t[3], QQ = t[4];
  const double bb = it == 0 ? rr : d.scal[AB_D2_BB];
  const double tol = d.scal[AB_D2_TOL];
  if (tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) {  // identical decision in every block and rank
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      d.scal[AB_D2_DONE] = 1.0;
      d.scal[AB_D2_RR] = rr;
      if (it == 0) d.scal[AB_D2_BB] = bb;
    }
    return;
  }
  const double alpha = PQ != 0.0 ? RR / PQ : 0.0;
  double rr_next = fma(alpha, fma(alpha, QQ, -2.0 * RQ), RR);
  if (rr_next < 0.0) rr_next = 0.0;
  const double beta = RR != 0.0 ? rr_next / RR : 0.0;
  const double2* rq_in = reinterpret_cast<const double2*>(d.rq[it & 1]);
  double2* rq_out = reinterpret_cast<double2*>(d.rq[(it + 1) & 1]);
  double2* xp = reinterpret_cast<double2*>(d.xp);
  const int R = d.tile_rows;
  double* zs = qs + R;
  const bool true_norm = tol > 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int64_t n_tiles = (d.n_rows + R - 1) / R;
  // persistent CTAs walk the tiles (the records are collected once per CTA)
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
  const int64_t row0 = tile * R;
  const int rows = (int)(d.n_rows - row0 < R ? d.n_rows - row0 : R);
  __syncthreads();  // the previous tile's shared-memory reads are done
  for (int li = threadIdx.x; li < rows; li += kD2Block) {
    const double2 v = rq_in[row0 + li];
    qs[li] = v.y;
    zs[li] = fma(-alpha, v.y, v.x);
  }
  const int g0 = d.tghost_ptr[tile], ng = d.tghost_ptr[tile + 1] - g0;
  for (int k = threadIdx.x; k < ng; k += kD2Block) {
    const double2 gv = rq_in[__ldg(d.tghost + g0 + k)];
    zs[R + k] = fma(-alpha, gv.y, gv.x);
  }
  __syncthreads();
  const int nsl = (rows + 31) >> 5;
  for (int sl = warp; sl < nsl; sl += kD2Block / 32) {
    const double az = sell_row_dot_smem<8>(d.slice_ptr + (row0 >> 5), d.tcols, d.vals, zs, sl, lane);
    const int li = sl * 32 + lane;
    if (li < rows) {
      const int64_t i = row0 + li;
      const double ri = zs[li];
      const double2 w = xp[i];
      const double pi = fma(beta, w.y, ri);
      xp[i] = make_double2(fma(alpha, w.y, w.x), pi);
      if (i < d.n_if) {
        d.tif[i] = az;
        for (int e = d.send_ptr[i]; e < d.send_ptr[i + 1]; ++e) d.peer_recv[d.send_peer[e]][d.send_off[e]] = az;
        rq_out[i] = make_double2(ri, qs[li]);  // q_{j-1} parked for k_d2_tile_iface
      } else {
        const double qi = fma(beta, qs[li], az);
        rq_out[i] = make_double2(ri, qi);
        v[0] += ri * ri;  // interior rows belong to this rank alone (own = 1)
        v[1] += true_norm ? ri * ri / d.dinv[i] : ri * ri;
        v[2] += pi * qi;
        v[3] += ri * qi;
        v[4] += qi * qi;
      }
    }
  }
  if (row0 < d.n_if) {  // a signalling tile: its puts are complete
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int q = 0; q < d.n_peers; ++q)
        if (d.peer_nsig[q] > 0) red_rel_u64(d.peer_cnt[q], 1ull);
    }
  }
  }
  double tot[5];
  if (grid_sum<5, kD2Block>(v, d.part, d.cnt, tot) && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) d.scal[AB_D2_INT + k] = tot[k];
    d.scal[AB_D2_BETA] = beta;
    d.scal[AB_D2_RR] = rr;
    if (it == 0) d.scal[AB_D2_BB] = bb;
  }
}

__global__ void __launch_bounds__(kD2Block) k_d2_tile_iface(ab_ddcg2_rank d) {
  __shared__ int sflag;
  if (d.scal[AB_D2_DONE] != 0.0) return;
  if (threadIdx.x == 0) sflag = 0;
  __syncthreads();
  const double hev = d.scal[AB_D2_HEV];
  if ((int)threadIdx.x < d.n_peers && d.peer_nsig[threadIdx.x] > 0) {
    const int q = d.peer_rank[threadIdx.x];
    const unsigned long long want = (unsigned long long)(hev + 1.0) * (unsigned long long)d.peer_nsig[threadIdx.x];
    const long long t0 = peer_time();
    while (ld_acq_u64(d.cnt_in + q) < want) {
      if (peer_time() - t0 > kPeerTimeoutNs) { sflag = 1; break; }
    }
  }
  __syncthreads();
  const bool failed = sflag != 0;
  const double beta = d.scal[AB_D2_BETA];
  const int it = (int)d.scal[AB_D2_IT];
  double2* rq_out = reinterpret_cast<double2*>(d.rq[(it + 1) & 1]);
  const double2* xp = reinterpret_cast<const double2*>(d.xp);
  const bool true_norm = d.scal[AB_D2_TOL] > 0.0;
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (!failed) {
    for (int64_t i = (int64_t)blockIdx.x * kD2Block + threadIdx.x; i < d.n_if; i += (int64_t)gridDim.x * kD2Block) {
      const double own_t = d.tif[i];
      double tsum = 0.0;
      bool mine = false;
      for (int e = d.recv_ptr[i]; e < d.recv_ptr[i + 1]; ++e) {
        if (!mine && d.recv_rank[e] > d.rank) { tsum += own_t; mine = true; }
        tsum += __ldcg(d.recv + d.recv_off[e]);
      }
      if (!mine) tsum += own_t;
      const double2 rv = rq_out[i];
      const double ri = rv.x;
      const double qi = fma(beta, rv.y, tsum);
      rq_out[i] = make_double2(ri, qi);
      const double pi = xp[i].y;
      const double w = d.own[i];
      v[0] += w * ri * ri;
      v[1] += true_norm ? w * ri * ri / d.dinv[i] : w * ri * ri;
      v[2] += w * pi * qi;
      v[3] += w * ri * qi;
      v[4] += w * qi * qi;
    }
  }
  double tot[5];
  double* part = d.part + d2_front_part(d.n_rows);
  uint32_t* cnt = d.cnt + d2_front_cnt(d.n_rows);
  if (grid_sum<5, kD2Block>(v, part, cnt, tot) && threadIdx.x == 0) {
    d.scal[AB_D2_HEV] = hev + 1.0;
    if (failed) {
      d.scal[AB_D2_FAIL] = 1.0;
      d.scal[AB_D2_DONE] = 1.0;
      return;
    }
    double rec[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) rec[k] = d.scal[AB_D2_INT + k] + tot[k];
    const double ep = d.scal[AB_D2_EPOCH] + 1.0;
    d.scal[AB_D2_EPOCH] = ep;
    d.scal[AB_D2_EPB] = ep;
    d.scal[AB_D2_IT] = (double)(it + 1);
    d2_publish<5>(d, (it + 1) & 1, rec, ep);
  }
}

// x' + alpha_K p (the x update of the last iteration, alpha from the last
// published record: every rank's totals, collected like the next iteration
// would) unless the solve converged; out[perm[i]] = s_i x'_i.
__global__ void __launch_bounds__(256) k_d2_finish_sp(ab_ddcg2_rank d, double* __restrict__ x_node) {
  __shared__ double sbuf[5 * 32];
  __shared__ int sflag;
  if (threadIdx.x == 0) sflag = 0;
  __syncthreads();
  double alpha = 0.0;
  if (d.scal[AB_D2_DONE] == 0.0 && d.scal[AB_D2_IT] > 0.0) {
    double t[5];
    if (d2_collect<5>(d, (int)d.scal[AB_D2_IT] & 1, d.scal[AB_D2_EPB], t, sbuf, &sflag))
      alpha = t[2] != 0.0 ? t[0] / t[2] : 0.0;
    else if (threadIdx.x == 0)
      d.scal[AB_D2_FAIL] = 1.0;
  }
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d.n_rows) {
    const double2 w = reinterpret_cast<const double2*>(d.xp)[i];
    x_node[d.perm[i]] = d.s[i] * fma(alpha, w.y, w.x);
  }
}

__global__ void k_d2_finish(ab_ddcg2_rank d, double* __restrict__ x_node) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d.n_rows) x_node[d.perm[i]] = d.scaled ? d.s[i] * d.x[i] : d.x[i];
}

}  // namespace ab

using namespace ab;

extern "C" {

int ab_peer_halo_grid(int32_t n_if) {
  const int g = (n_if + kPeerBlock - 1) / kPeerBlock;
  return g < 1 ? 1 : (g > 64 ? 64 : g);
}

static int check_halo(const ab_peer_halo* h, int ncomp, int stride, const char* what) {
  if (!h || !h->state || !h->recv || !h->cnt_in) return fail(what);
  if (ncomp < 1 || ncomp > 3 || stride < ncomp) return fail("peer halo: ncomp must be 1..3 and <= stride");
  if (h->n_nbr < 0 || h->n_nbr > AB_PEER_MAX) return fail("peer halo: too many neighbours");
  if (h->n_cta != ab_peer_halo_grid(h->n_if)) return fail("peer halo: n_cta != ab_peer_halo_grid(n_if)");
  return AB_OK;
}

int ab_peer_halo_put(const ab_peer_halo* h, const double* field, int32_t ncomp, int32_t stride, void* stream) {
  if (int rc = check_halo(h, ncomp, stride, "ab_peer_halo_put: incomplete descriptor")) return rc;
  k_halo_put<<<h->n_cta, kPeerBlock, 0, S(stream)>>>(*h, field, ncomp, stride);
  return check_launch("ab_peer_halo_put");
}

int ab_peer_halo_add(const ab_peer_halo* h, double* field, int32_t ncomp, int32_t stride, void* stream) {
  if (int rc = check_halo(h, ncomp, stride, "ab_peer_halo_add: incomplete descriptor")) return rc;
  k_halo_add<<<h->n_cta, kPeerBlock, 0, S(stream)>>>(*h, field, ncomp, stride);
  return check_launch("ab_peer_halo_add");
}

int64_t ab_ddcg2_part_size(int64_t n_rows) {
  // front (row-parallel kernels) + the interface kernels' (5 values over <= kD2IfGrid blocks)
  return d2_front_part(n_rows) + 5 * (kD2IfGrid + 4) + 8;
}

static int check_d2(const ab_ddcg2_rank* d, const char* what) {
  if (!d || !d->slice_ptr || !d->scal || !d->part || !d->cnt || !d->rec) return fail(what);
  if (d->n_peers < 0 || d->n_peers > AB_PEER_MAX || d->n_ranks > 32) return fail("ddcg2: at most 8 peers / 32 ranks");
  return AB_OK;
}

static int check_sp(const ab_ddcg2_rank* d, const char* what) {
  if (!d->scaled || d->tile_rows <= 0 || !d->xp || !d->rq[0] || !d->rq[1] || !d->s)
    return fail(what);
  if ((((uintptr_t)d->xp) | ((uintptr_t)d->rq[0]) | ((uintptr_t)d->rq[1])) & 15)
    return fail("ddcg2 single pass: xp, rq must be 16-byte aligned");
  return AB_OK;
}

int ab_ddcg2_init(const ab_ddcg2_rank* d, const double* b, double* b_zero, double tol, void* stream) {
  if (int rc = check_d2(d, "ab_ddcg2_init: incomplete descriptor")) return rc;
  const unsigned g = grid_for(d->n_rows, kD2Block);
  if (d->single_pass) {
    if (int rc = check_sp(d, "ab_ddcg2_init: single pass needs the scaled form, a tile map, xp and rq")) return rc;
    k_d2_init_sp<<<g > 0 ? g : 1, kD2Block, 0, S(stream)>>>(*d, b, tol);
    if (int rc = check_launch("ab_ddcg2_init")) return rc;
    if (b_zero && d->n_rows > 0) k_d2_zero<<<grid_for(d->n_rows, 256), 256, 0, S(stream)>>>(d->n_rows, b_zero);
    return check_launch("ab_ddcg2_init");
  }
  k_d2_init<<<g > 0 ? g : 1, kD2Block, 0, S(stream)>>>(*d, b, b_zero, tol);
  if (int rc = check_launch("ab_ddcg2_init")) return rc;
  if (b_zero && d->n_rows > 0) k_d2_zero<<<grid_for(d->n_rows, 256), 256, 0, S(stream)>>>(d->n_rows, b_zero);
  return check_launch("ab_ddcg2_init");
}

int ab_ddcg2_spmv(const ab_ddcg2_rank* d, void* stream) {
  if (int rc = check_d2(d, "ab_ddcg2_spmv: incomplete descriptor")) return rc;
  if (d->tile_rows > 0) {
    const int64_t R = d->tile_rows;
    if (R % 64 || !d->tcols || !d->tghost_ptr || !d->tghost || R + d->tmax_ghost > 65536)
      return fail("ab_ddcg2_spmv: bad tile map (tile_rows % 64, tcols, tghost_ptr, tghost, R + max ghost <= 65536)");
    if (d->nsig != (int32_t)((d->n_if + R - 1) / R)) return fail("ab_ddcg2_spmv: nsig must count tiles when tiled");
    const size_t smem = (size_t)(R + d->tmax_ghost) * sizeof(double);
    static size_t smem_set = 0;
    if (smem > 48 * 1024 && smem > smem_set) {
      if (cudaFuncSetAttribute(k_d2_spmv_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return fail("ab_ddcg2_spmv: shared memory request rejected (tile too large)");
      smem_set = smem;
    }
    const unsigned g = (unsigned)((d->n_rows + R - 1) / R);
    k_d2_spmv_tile<<<g > 0 ? g : 1, kD2Block, smem, S(stream)>>>(*d);
    return check_launch("ab_ddcg2_spmv");
  }
  const unsigned g = grid_for(d->n_rows, kD2Block);
  k_d2_spmv<<<g > 0 ? g : 1, kD2Block, 0, S(stream)>>>(*d);
  return check_launch("ab_ddcg2_spmv");
}

int ab_ddcg2_iface(const ab_ddcg2_rank* d, void* stream) {
  if (int rc = check_d2(d, "ab_ddcg2_iface: incomplete descriptor")) return rc;
  int g = (int)((d->n_if + kD2Block - 1) / kD2Block);
  if (g < 1) g = 1;
  if (g > kD2IfGrid) g = kD2IfGrid;
  k_d2_iface<<<g, kD2Block, 0, S(stream)>>>(*d);
  return check_launch("ab_ddcg2_iface");
}

int ab_ddcg2_update(const ab_ddcg2_rank* d, void* stream) {
  if (int rc = check_d2(d, "ab_ddcg2_update: incomplete descriptor")) return rc;
  unsigned g = grid_for((d->n_rows + 1) / 2, kD2Block);
  if (g > 148u * 8u) g = 148u * 8u;  // grid-stride: 8 CTAs per SM
  k_d2_update<<<g > 0 ? g : 1, kD2Block, 0, S(stream)>>>(*d);
  return check_launch("ab_ddcg2_update");
}

int ab_ddcg2_tile_iter(const ab_ddcg2_rank* d, void* stream) {
  if (int rc = check_d2(d, "ab_ddcg2_tile_iter: incomplete descriptor")) return rc;
  if (int rc = check_sp(d, "ab_ddcg2_tile_iter: needs single_pass, the scaled form, a tile map, xp and rq")) return rc;
  if (!d->single_pass) return fail("ab_ddcg2_tile_iter: descriptor not in single-pass mode");
  const int64_t R = d->tile_rows;
  if (R % 64 || !d->tcols || !d->tghost_ptr || !d->tghost || R + d->tmax_ghost > 65536)
    return fail("ab_ddcg2_tile_iter: bad tile map");
  if (d->nsig != (int32_t)((d->n_if + R - 1) / R)) return fail("ab_ddcg2_tile_iter: nsig must count tiles");
  const size_t smem = (size_t)(2 * R + d->tmax_ghost) * sizeof(double);
  static size_t smem_set = 0;
  if (smem > 48 * 1024 && smem > smem_set) {
    if (cudaFuncSetAttribute(k_d2_tile_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return fail("ab_ddcg2_tile_iter: shared memory request rejected (tile too large)");
    smem_set = smem;
  }
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_d2_tile_iter, kD2Block, smem);
    if (per_sm < 1) per_sm = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t g = (d->n_rows + R - 1) / R;
  if (g > (int64_t)sms * per_sm) g = (int64_t)sms * per_sm;
  k_d2_tile_iter<<<(unsigned)(g > 0 ? g : 1), kD2Block, smem, S(stream)>>>(*d);
  return check_launch("ab_ddcg2_tile_iter");
}

int ab_ddcg2_tile_iface(const ab_ddcg2_rank* d, void* stream) {
  if (int rc = check_d2(d, "ab_ddcg2_tile_iface: incomplete descriptor")) return rc;
  if (!d->single_pass) return fail("ab_ddcg2_tile_iface: descriptor not in single-pass mode");
  int g = (int)((d->n_if + kD2Block - 1) / kD2Block);
  if (g < 1) g = 1;
  if (g > kD2IfGrid) g = kD2IfGrid;
  k_d2_tile_iface<<<g, kD2Block, 0, S(stream)>>>(*d);
  return check_launch("ab_ddcg2_tile_iface");
}

int ab_ddcg2_finish(const ab_ddcg2_rank* d, double* x_node, void* stream) {
  if (int rc = check_d2(d, "ab_ddcg2_finish: incomplete descriptor")) return rc;
  if (d->single_pass) {
    if (d->n_rows > 0) k_d2_finish_sp<<<grid_for(d->n_rows, 256), 256, 0, S(stream)>>>(*d, x_node);
    return check_launch("ab_ddcg2_finish");
  }
  if (d->n_rows > 0) k_d2_finish<<<grid_for(d->n_rows, 256), 256, 0, S(stream)>>>(*d, x_node);
  return check_launch("ab_ddcg2_finish");
}

}  // extern "C"
