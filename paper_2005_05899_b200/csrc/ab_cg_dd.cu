// Resident Jacobi-PCG of a decomposed domain, fused with its interface
// exchange (include/alyab200.h "K5 across ranks").
//
// The element-disjoint decomposition duplicates interface nodes
// (PAPER.md:325-330): each rank's Laplacian rows at interface nodes hold only
// that rank's elements, so (A z)_i = sum over the sharing ranks of their
// partial products, and the dots weight every node once (own = 1 on its
// lowest rank).  Per iteration, without leaving the kernel:
//   ghost gather   z of the CTA's remote columns -> shared memory (own rank)
//   SpMV           t = A_r z per row; interface rows write t straight into
//                  every sharing rank's receive array (peer memory);
//                  p = z + beta p, q = t + beta q (interface rows: partial)
//   signal/wait    per-CTA release-add on each peer's arrival counter, then
//                  acquire-poll of this rank's counters (monotone over the run)
//   interface add  q_i += received partials (ascending peer rank), p.q
//   reduce A       CTAs: grid barrier + ordered all-sum; ranks: {value, epoch}
//                  records into every rank's slots, summed in rank order
//   update         x += alpha p, r -= alpha q, z = D^-1 r, r.z, r.r
//   reduce B       as A; also publishes z to the rank's CTAs
// Every rank sums the same numbers in the same order, so all ranks take the
// same alpha, beta and stopping decision.  Peer waits time out (10 s) by
// setting red[ITERS] = -1 instead of hanging the device.
#include <cstring>

#include "ab_cg_common.cuh"

namespace ab {

static_assert(sizeof(ab_cg_dd_rank) == 536, "ab_cg_dd_rank layout (mirrored by ddcg.AbCgDdRank)");
constexpr int kDdRowsPerThread = 8;
constexpr long long kDdTimeoutNs = 10000000000ll;

__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acq_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// {value, epoch} record: the value is stored first (relaxed), then the
// epoch word with release semantics; a reader acquires the epoch and only
// then loads the value, so a matching epoch always comes with its value (a
// 16-byte vector access is not single-copy atomic).  A slot is rewritten
// only after every rank has consumed it (the next write of a set needs the
// other set's records of every rank, published after their collection).
__device__ __forceinline__ void st_rec_sys(double* p, double v, double e) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
  asm volatile("st.release.sys.global.f64 [%0], %1;" ::"l"(p + 1), "d"(e) : "memory");
}
__device__ __forceinline__ double ld_rec_epoch(const double* p) {
  double e;
  asm volatile("ld.acquire.sys.global.f64 %0, [%1];" : "=d"(e) : "l"(p + 1) : "memory");
  return e;
}
__device__ __forceinline__ double ld_rec_value(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Rank-wide failure flag (bar[1], zeroed per solve): a CTA whose peer wait
// times out raises it; grid barriers give up when it is set and every CTA
// leaves the iteration loop after the next barrier, so no CTA is left
// spinning in a barrier its siblings will never reach.
__device__ __forceinline__ void raise_failure(unsigned* bar) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
}
__device__ __forceinline__ unsigned failure_flag(unsigned* bar) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
  return v;
}
__device__ __forceinline__ void dd_grid_barrier(unsigned* bar, unsigned target, int* s_failed) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      if (failure_flag(bar)) { *s_failed = 1; break; }
    }
    if (failure_flag(bar)) *s_failed = 1;
  }
  __syncthreads();
}

struct DdCtx {
  const ab_cg_dd_rank* g;
  int lcta;          // CTA index within the rank
  int nb;            // CTAs of the rank
  int* failed;       // shared flag
};

// Cross-CTA part of a reduction: NV block-reduced values (valid in thread
// 0) -> grid barrier on g.bar -> ordered rank total `loc` in every thread;
// with several ranks the total is published as {value, epoch} records into
// every rank's slot set `set`.
template <int NV>
__device__ __forceinline__ void dd_publish(const DdCtx& c, double (&v)[NV], int set, double ep, unsigned& nbar,
                                           double* sred, double* bcast, double (&loc)[NV]) {
  const ab_cg_dd_rank& g = *c.g;
  double* part = g.part + (size_t)set * 2 * c.nb;
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) part[(size_t)k * c.nb + c.lcta] = v[k];
  dd_grid_barrier(g.bar, ++nbar * (unsigned)c.nb, c.failed);
  all_sum_par<NV>(part, c.nb, sred, bcast, loc);
  const int P = g.n_ranks;
  if (P > 1 && c.lcta == 0 && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const size_t o = (((size_t)set * P + g.rank) * 2 + k) * 2;
      st_rec_sys(g.red_in + o, loc[k], ep);
      for (int q = 0; q < g.n_peers; ++q) st_rec_sys(g.peer_red[q] + o, loc[k], ep);
    }
  }
}

// Cross-rank part: thread q polls rank q's record (local memory), then the
// totals are summed in rank order (identical on every rank).
template <int NV>
__device__ __forceinline__ void dd_collect(const DdCtx& c, int set, double ep, double* bcast, const double (&loc)[NV],
                                           double (&out)[NV]) {
  const ab_cg_dd_rank& g = *c.g;
  const int P = g.n_ranks;
  if (P == 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = loc[k];
    return;
  }
  double w[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) w[k] = 0.0;
  if ((int)threadIdx.x < P) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double* rec = g.red_in + (((size_t)set * P + threadIdx.x) * 2 + k) * 2;
      double val = 0.0;
      const long long tw = gtime();  // timeout per wait
      for (;;) {
        if (ld_rec_epoch(rec) == ep) { val = ld_rec_value(rec); break; }
        if (*c.failed || gtime() - tw > kDdTimeoutNs) {
          *c.failed = 1;
          raise_failure(g.bar);
          break;
        }
      }
      w[k] = val;
    }
  }
  __syncthreads();  // bcast of the previous use has been read
  if (threadIdx.x < 32) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double acc = 0.0;
      for (int q = 0; q < P; ++q) acc += __shfl_sync(0xffffffffu, w[k], q);
      if (threadIdx.x == 0) bcast[k] = acc;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = bcast[k];
  __syncthreads();
}

__global__ void __launch_bounds__(kResBlock, 1) k_cg_dd(const ab_cg_dd_rank* __restrict__ groups, int n_groups,
                                                        int maxit, double tol) {
  extern __shared__ double smem[];
  __shared__ double sred[2 * (kResBlock / 32)];
  __shared__ double bcast[4];
  __shared__ int s_failed;
  __shared__ ab_cg_dd_rank s_g;  // the rank's descriptor, read with LDS from here on
  __shared__ uint32_t s_taddr;
  // ---- which rank (group) this CTA works for
  int gi = 0;
  while (gi + 1 < n_groups && (int)blockIdx.x >= groups[gi + 1].cta0) ++gi;
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(groups + gi);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&s_g);
    for (int k = threadIdx.x; k < (int)(sizeof(ab_cg_dd_rank) / 4); k += kResBlock) dst[k] = src[k];
    __syncthreads();
  }
  const ab_cg_dd_rank& g = s_g;
  const int lcta = (int)blockIdx.x - g.cta0;
  if (threadIdx.x == 0) s_failed = 0;
  DdCtx c{&g, lcta, g.n_cta, &s_failed};
  const int64_t n = g.n_rows;
  const int64_t RB = g.rows_per_cta;
  const int64_t r0 = (int64_t)lcta * RB;
  const int64_t r1 = r0 + RB < n ? r0 + RB : n;
  const int nloc = r1 > r0 ? (int)(r1 - r0) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsl = (nloc + 31) >> 5;
  const int64_t s_first = r0 >> 5;
  const int g0 = g.ghost_ptr[lcta];
  const int ng = g.ghost_ptr[lcta + 1] - g0;
  double* sr = smem;
  double* spp = sr + RB;
  double* sq = spp + RB;
  double* sz = sq + RB;  // [RB] own rows, then ghosts
  // x lives in tensor memory: thread (warp w, lane) keeps x of its phase-B
  // rows l = threadIdx.x + k * kResBlock in columns 2k, 2k + 1 of its lane
  // (warp w's 32-lane quarter, 64-column slice of its warp group)
  const uint32_t taddr = tmem_alloc_all(&s_taddr);
  const uint32_t tx = taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
  // shared tables: interface bits, ownership bits, slice pointers, ghost ids
  uint32_t* smask = reinterpret_cast<uint32_t*>(sz + RB + g.max_ghost);  // [RB / 32]
  uint32_t* sown = smask + RB / 32;                                       // [RB / 32]
  int64_t* tsp_s = reinterpret_cast<int64_t*>(sown + RB / 32);                  // [RB / 32 + 1], 8-aligned
  int32_t* tg_s = reinterpret_cast<int32_t*>(tsp_s + RB / 32 + 1);        // [max_ghost]
  const int64_t* tsp = tsp_s;
  const int32_t* tg = tg_s;
  const uint16_t* lcol = g.cols;
  const double* sval = g.vals;
  const int P = g.n_ranks;
  const unsigned long long hbase = g.evbase[0];
  const double ebase = (double)g.evbase[1];
  double ep = ebase;
  unsigned nbar = 0;
  for (int k = threadIdx.x; k < nsl; k += kResBlock) smask[k] = g.ifmask[(r0 >> 5) + k];
  for (int k = threadIdx.x; k <= nsl; k += kResBlock) tsp_s[k] = g.slice_ptr[s_first + k];
  for (int k = threadIdx.x; k < ng; k += kResBlock) tg_s[k] = g.ghost[g0 + k];
  for (int k = threadIdx.x; k < nsl; k += kResBlock) {  // own[] is 0/1: one bit per row
    uint32_t w = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t i = r0 + 32 * k + b;
      if (i < n && g.own[i] != 0.0) w |= 1u << b;
    }
    sown[k] = w;
  }
  __syncthreads();
  const int ri0 = g.rrow_ptr[lcta], ri1 = g.rrow_ptr[lcta + 1];

  // ---- init: r = b (fixed rows 0), z = D^-1 r, x = p = q = 0
  double a0 = 0.0, a1 = 0.0;
  for (int l = threadIdx.x; l < nloc; l += kResBlock) {
    const int64_t i = r0 + l;
    const int64_t ni = g.perm[i];
    double ri = g.b_in[ni];
    if (g.fixed && g.fixed[i]) ri = 0.0;
    if (g.b_zero) g.b_zero[ni] = 0.0;
    const double zi = g.dinv[i] * ri;
    sr[l] = ri; sz[l] = zi; spp[l] = 0.0; sq[l] = 0.0;
    g.zg[i] = zi;
    if ((sown[l >> 5] >> (l & 31)) & 1u) {
      a0 += ri * zi;
      a1 += ri * ri;
    }
  }
#pragma unroll
  for (int k = 0; k < kDdRowsPerThread; ++k) tm_st(tx + 2 * k, 0.0);
  tm_wait_st();
  double t2[2], l2[2];
  {
    double v[2] = {a0, a1};
    block_sum<2, kResBlock>(v, sred);
    ep += 1.0;
    dd_publish<2>(c, v, 0, ep, nbar, sred, bcast, l2);
    dd_collect<2>(c, 0, ep, bcast, l2, t2);
  }
  double rz = t2[0], rr = t2[1];
  const double bb = rr;
  double rz_old = 0.0;
  int it = 0;
  // The r.z / r.r records of iteration i are collected only after the SpMV
  // of iteration i + 1 has been computed and shipped (that SpMV needs z,
  // not beta): the cross-rank wait of reduction B overlaps the matrix
  // stream.  A(z) per row waits in TMEM (columns 16 + 2k) for beta.
  bool pending = false;
  double epB = 0.0;
  unsigned long long hev = 0;  // halo events of this solve
  for (; it < maxit; ++it) {
    if (s_failed) break;
    if (threadIdx.x == 0 && failure_flag(g.bar)) s_failed = 1;
    __syncthreads();
    if (s_failed) break;
    if (!pending && tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) break;
    for (int k = threadIdx.x; k < ng; k += kResBlock) sz[RB + k] = __ldcg(g.zg + tg[k]);
    __syncthreads();
    // ---- SpMV: A z per row -> TMEM; interface rows ship it to the sharers
#pragma unroll 1
    for (int k = 0; k * (kResBlock / 32) + warp < nsl; ++k) {
      const int sl = warp + k * (kResBlock / 32);
      const double az = sell_row_dot_smem<kLocChunk>(tsp, lcol, sval, sz, sl, lane);
      tm_st(tx + 16 + 2 * k, az);
      const int l = sl * 32 + lane;
      if (l < nloc && ((smask[sl] >> lane) & 1u)) {
        const int64_t i = r0 + l;
        for (int e = g.send_ptr[i]; e < g.send_ptr[i + 1]; ++e) g.peer_recv[g.send_peer[e]][g.send_off[e]] = az;
      }
    }
    ++hev;
    if (P > 1) {  // this CTA's sends are complete -> one arrival on every peer's counter
      __syncthreads();
      if (threadIdx.x == 0) {
        if (g.pad0_) __threadfence(); else __threadfence_system();  // pad0_ = 1: every peer on this device
        for (int q = 0; q < g.n_peers; ++q) red_rel_sys_u64(g.peer_cnt[q], 1ull);
      }
    }
    if (pending) {  // reduction B of the previous iteration
      dd_collect<2>(c, 2, epB, bcast, l2, t2);
      rz_old = rz;
      rz = t2[0];
      rr = t2[1];
      pending = false;
      if (tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) break;
    }
    const double beta = rz_old != 0.0 ? rz / rz_old : 0.0;
    if (P > 1) {  // every CTA of every peer has shipped (monotone counters)
      if ((int)threadIdx.x < g.n_peers) {
        const int q = g.peer_rank[threadIdx.x];
        const unsigned long long want = (hbase + hev) * (unsigned long long)g.peer_ncta[threadIdx.x];
        const long long tw = gtime();
        while (ld_acq_sys_u64(g.cnt_in + q) < want) {
          if (s_failed || gtime() - tw > kDdTimeoutNs) {
            s_failed = 1;
            raise_failure(g.bar);
            break;
          }
        }
      }
    }
    tm_wait_st();
    __syncthreads();
    // ---- p = z + beta p, q = A z + beta q (+ neighbours' partials), p.q
    double pq = 0.0;
#pragma unroll 1
    for (int k = 0; k * (kResBlock / 32) + warp < nsl; ++k) {
      const int sl = warp + k * (kResBlock / 32);
      uint32_t lo, hi;
      tm_ld(tx + 16 + 2 * k, lo, hi);
      tm_wait_ld();
      const double az = tm_val(lo, hi);
      const int l = sl * 32 + lane;
      if (l < nloc) {
        const double p = fma(beta, spp[l], sz[l]);
        double q;
        if ((smask[sl] >> lane) & 1u) {
          const int64_t i = r0 + l;
          // rrow is ascending: find this row's receive range
          int lo_k = ri0, hi_k = ri1 - 1;
          while (lo_k < hi_k) {
            const int mid = (lo_k + hi_k) >> 1;
            if (g.rrow[mid] < i) lo_k = mid + 1; else hi_k = mid;
          }
          // (A z)_i = sum of the sharing ranks' partials in global rank
          // order, this rank's at its position: every rank forms the same
          // bits, so duplicated interface values stay identical
          double t = 0.0;
          bool own_added = false;
          for (int e = g.recv_ptr[lo_k]; e < g.recv_ptr[lo_k + 1]; ++e) {
            const int off = g.recv_off[e];
            if (!own_added && off / g.recv_stride > g.rank) { t += az; own_added = true; }
            t += __ldcg(g.recv + off);
          }
          if (!own_added) t += az;
          q = fma(beta, sq[l], t);
          if ((sown[sl] >> lane) & 1u) pq += p * q;
        } else {
          q = fma(beta, sq[l], az);
          pq += p * q;  // non-interface rows are owned
        }
        spp[l] = p;
        sq[l] = q;
      }
    }
    // D^-1 of this thread's update rows: in flight across reduction A
    double dv[kDdRowsPerThread];
#pragma unroll
    for (int k = 0; k < kDdRowsPerThread; ++k) {
      const int l = threadIdx.x + k * kResBlock;
      dv[k] = l < nloc ? __ldg(g.dinv + r0 + l) : 0.0;
    }
    double t1[1], l1[1];
    {
      double v[1] = {pq};
      block_sum<1, kResBlock>(v, sred);
      ep += 1.0;
      dd_publish<1>(c, v, 1, ep, nbar, sred, bcast, l1);
      dd_collect<1>(c, 1, ep, bcast, l1, t1);
    }
    const double alpha = t1[0] != 0.0 ? rz / t1[0] : 0.0;
    // ---- x += alpha p, r -= alpha q, z = D^-1 r
    double b0 = 0.0, b1 = 0.0;
    uint32_t xw[kDdRowsPerThread][2];
#pragma unroll
    for (int k = 0; k < kDdRowsPerThread; ++k) tm_ld(tx + 2 * k, xw[k][0], xw[k][1]);
    tm_wait_ld();
#pragma unroll
    for (int k = 0; k < kDdRowsPerThread; ++k) {
      const int l = threadIdx.x + k * kResBlock;
      const double xo = tm_val(xw[k][0], xw[k][1]);
      tm_st(tx + 2 * k, l < nloc ? fma(alpha, spp[l], xo) : xo);
      if (l < nloc) {
        const double ri = fma(-alpha, sq[l], sr[l]);
        const double zi = dv[k] * ri;
        sr[l] = ri;
        sz[l] = zi;
        g.zg[r0 + l] = zi;
        if ((sown[l >> 5] >> (l & 31)) & 1u) {
          b0 += ri * zi;
          b1 += ri * ri;
        }
      }
    }
    {
      double v[2] = {b0, b1};
      block_sum<2, kResBlock>(v, sred);
      ep += 1.0;
      epB = ep;
      dd_publish<2>(c, v, 2, ep, nbar, sred, bcast, l2);  // local grid barrier: z published in the rank
      pending = true;
    }
  }
  if (pending) {
    dd_collect<2>(c, 2, epB, bcast, l2, t2);
    rz_old = rz;
    rz = t2[0];
    rr = t2[1];
  }
  tm_wait_st();
#pragma unroll
  for (int k = 0; k < kDdRowsPerThread; ++k) {
    uint32_t lo, hi;
    tm_ld(tx + 2 * k, lo, hi);
    tm_wait_ld();
    const int l = threadIdx.x + k * kResBlock;
    if (l < nloc) g.x_out[g.perm[r0 + l]] = tm_val(lo, hi);
  }
  tmem_free_all(taddr);
  // every CTA of the rank has read evbase before its first reduction
  if (lcta == 0 && threadIdx.x == 0) {
    g.red[AB_RED_RZN] = rz;
    g.red[AB_RED_RR] = rr;
    g.red[AB_RED_ITERS] = s_failed ? -1.0 : (double)it;
    if (s_failed) g.red[AB_RED_FAIL] = 1.0;  // sticky until the host clears it
    g.sc[AB_SC_BB] = bb;
    g.evbase[0] = hbase + hev;
    g.evbase[1] = (unsigned long long)ep;
  }
}

}  // namespace ab

using namespace ab;

extern "C" {

int ab_cg_dd(const ab_cg_dd_rank* groups_dev, int32_t n_groups, int32_t n_cta_total, int32_t maxit, double tol,
             int64_t max_rows_per_cta, int32_t max_ghost, void* stream) {
  if (!groups_dev || n_groups <= 0 || n_cta_total <= 0) return fail("ab_cg_dd: empty launch");
  if (max_rows_per_cta > (int64_t)kDdRowsPerThread * kResBlock || max_rows_per_cta % 32)
    return fail("ab_cg_dd: rows per CTA must be a multiple of 32 and <= 8192");
  int dev = 0, optin = 0, coop = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (!coop) return fail("ab_cg_dd: cooperative launch unsupported");
  if (n_cta_total > sms) return fail("ab_cg_dd: more CTAs than SMs");
  const size_t smem = (size_t)(4 * max_rows_per_cta + max_ghost) * 8 + (size_t)(max_rows_per_cta / 32 + 1) * 8 +
                      (size_t)(max_rows_per_cta / 32 + 1) * 8 + (size_t)max_ghost * 4 + 16;
  if (smem + 1024 > (size_t)optin) return fail("ab_cg_dd: rows + ghosts do not fit in shared memory");
  if (cudaFuncSetAttribute((const void*)k_cg_dd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return fail("ab_cg_dd: cannot reserve shared memory");
  int ng = n_groups, mi = maxit;
  void* args[] = {(void*)&groups_dev, &ng, &mi, &tol};
  cudaError_t e =
      cudaLaunchCooperativeKernel((const void*)k_cg_dd, dim3(n_cta_total), dim3(kResBlock), args, smem, S(stream));
  if (e != cudaSuccess) {
    set_error(std::string("ab_cg_dd: ") + cudaGetErrorString(e));
    return AB_ECUDA;
  }
  return check_launch("ab_cg_dd");
}

int ab_ipc_get_handle(const void* dev_ptr, unsigned char* handle64, int64_t* offset) {
  if (!dev_ptr || !handle64 || !offset) return fail("ab_ipc_get_handle: null argument");
  // the handle names the whole allocation: report dev_ptr's offset in it
  // (pool allocators hand out pieces of larger blocks)
  typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
    return fail("ab_ipc_get_handle: cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (reinterpret_cast<GetRange>(fn)(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
    return fail("ab_ipc_get_handle: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) {
    set_error(std::string("ab_ipc_get_handle: ") + cudaGetErrorString(e));
    return AB_ECUDA;
  }
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, 64);
  *offset = (int64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  return AB_OK;
}

int ab_ipc_open_handle(const unsigned char* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail("ab_ipc_open_handle: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error(std::string("ab_ipc_open_handle: ") + cudaGetErrorString(e));
    return AB_ECUDA;
  }
  return AB_OK;
}

int ab_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return AB_OK;
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) {
    set_error(std::string("ab_ipc_close: ") + cudaGetErrorString(e));
    return AB_ECUDA;
  }
  return AB_OK;
}

}  // extern "C"
