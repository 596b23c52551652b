// Rejected resident-CG variants (measured slower than k_cg_resident_local on C2,
// DESIGN.md §4), kept here for the record.  NOT compiled into libalyab200.so; they
// reference helpers of paper_2005_05899_b200/csrc/ab_cg_common.cuh and ab_solver.cu.
// Extracted from ab_solver.cu at round 1 end.

// ---------------------------------------------------------------------------
// Resident CG: the whole solve in ONE cooperative kernel (one CTA per SM).
// Every CTA owns a contiguous, slice-aligned range of rows and keeps their
// x, r, z, p and q in shared memory for all iterations (D^-1 is re-read from
// L2 in phase B); only z goes to global memory, for the neighbours' gathers.
// Per iteration the matrix is streamed (the next slice of every warp is
// bulk-prefetched into L2 by the TMA engine while the current one is
// gathered) and the two grid-wide reductions are deterministic (per-CTA
// partials, summed in index order by every CTA after a grid barrier).
// Convergence (tol > 0) is tested on the device, identically in all CTAs.
// Used when the owned rows fit in shared memory (C2: 4768 rows x 40 B per
// SM); otherwise the kernels above run.  Launched cooperatively so that all
// CTAs are co-resident for the grid barriers.
// ---------------------------------------------------------------------------

// Bulk prefetch of one SELL slice (column indices + values) into L2.
__device__ __forceinline__ void prefetch_slice(const int64_t* __restrict__ sp, const int32_t* scol,
                                               const double* sval, int64_t s) {
  const int64_t b = sp[s];
  const uint32_t cnt = (uint32_t)(sp[s + 1] - b);
  if (cnt == 0) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(scol + b), "r"(cnt * 4u) : "memory");
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sval + b), "r"(cnt * 8u) : "memory");
}

// Ordered sum of nb per-CTA partials (layout part[k*nb+b]); identical in
// every CTA, broadcast through shared memory.
template <int NV>
__device__ __forceinline__ void all_sum(const double* part, int nb, double* bcast, double (&out)[NV]) {
  if (threadIdx.x < 32) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double acc = 0.0;
      for (int b = threadIdx.x; b < nb; b += 32) acc += __ldcg(part + (size_t)k * nb + b);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (threadIdx.x == 0) bcast[k] = acc;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = bcast[k];
  __syncthreads();
}

__global__ void __launch_bounds__(kResBlock, 1) k_cg_resident(
    int64_t n, int64_t rows_per_cta, const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
    const double* __restrict__ sval, const double* __restrict__ b_in, double* b_zero, const uint8_t* __restrict__ fixed,
    const double* __restrict__ dinv, double* __restrict__ x_out, double* zg, int maxit, double tol, double* red,
    double* sc, double* part, unsigned* bar) {
  unsigned nbar = 0;
  extern __shared__ double smem[];
  __shared__ double sred[2 * (kResBlock / 32)];
  __shared__ double bcast[4];
  const int nb = gridDim.x;
  const int64_t RB = rows_per_cta;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int64_t r1 = r0 + RB < n ? r0 + RB : n;
  const int nloc = r1 > r0 ? (int)(r1 - r0) : 0;
  double* sx = smem;
  double* sr = sx + RB;
  double* sz = sr + RB;
  double* spp = sz + RB;
  double* sq = spp + RB;
  double* partA = part;                   // [nb]     p.q
  double* partB = part + nb;              // [2][nb]  r.z, r.r
  double* partI = part + 3 * (size_t)nb;  // [2][nb]  init r.z, r.r
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsl = (nloc + 31) >> 5;
  const int64_t s_first = r0 >> 5;  // r0 is slice aligned

  double a0 = 0.0, a1 = 0.0;
  for (int l = threadIdx.x; l < nloc; l += kResBlock) {
    const int64_t i = r0 + l;
    double ri = b_in[i];
    if (fixed && fixed[i]) ri = 0.0;
    if (b_zero) b_zero[i] = 0.0;
    const double zi = dinv[i] * ri;
    sx[l] = 0.0; sr[l] = ri; sz[l] = zi; spp[l] = 0.0; sq[l] = 0.0;
    zg[i] = zi;
    a0 += ri * zi;
    a1 += ri * ri;
  }
  {
    double v[2] = {a0, a1};
    block_sum<2, kResBlock>(v, sred);
    if (threadIdx.x == 0) { partI[blockIdx.x] = v[0]; partI[nb + blockIdx.x] = v[1]; }
  }
  grid_barrier(bar, ++nbar * nb);
  double t2[2];
  all_sum<2>(partI, nb, bcast, t2);
  double rz = t2[0], rr = t2[1];
  const double bb = rr;
  double rz_old = 0.0;
  int it = 0;
  for (; it < maxit; ++it) {
    if (tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) break;  // same test as the host path
    const double beta = rz_old != 0.0 ? rz / rz_old : 0.0;
    // ---- phase A: p = z + beta p; q = A z + beta q
    double pq = 0.0;
    if (it == 0 && lane == 0 && warp < nsl) prefetch_slice(sp, scol, sval, s_first + warp);
#pragma unroll 1
    for (int sl = warp; sl < nsl; sl += kResBlock / 32) {
      const int64_t s = s_first + sl;
      // the TMA engine pulls the warp's next slice into L2 meanwhile
      if (lane == 0 && sl + kResBlock / 32 < nsl) prefetch_slice(sp, scol, sval, s + kResBlock / 32);
      const double az = sell_row_dot<true>(sp, scol, sval, zg, s * 32 + lane);
      const int l = sl * 32 + lane;
      if (l < nloc) {
        const double p = fma(beta, spp[l], sz[l]);
        const double q = fma(beta, sq[l], az);
        spp[l] = p;
        sq[l] = q;
        pq += p * q;
      }
    }
    {
      double v[1] = {pq};
      block_sum<1, kResBlock>(v, sred);
      if (threadIdx.x == 0) partA[blockIdx.x] = v[0];
    }
    grid_barrier(bar, ++nbar * nb);  // all gathers of z done, p.q partials visible
    double t1[1];
    all_sum<1>(partA, nb, bcast, t1);
    const double alpha = t1[0] != 0.0 ? rz / t1[0] : 0.0;
    // ---- phase B: x += alpha p, r -= alpha q, z = D^-1 r
    if (lane == 0 && it + 1 < maxit && warp < nsl) prefetch_slice(sp, scol, sval, s_first + warp);
    double b0 = 0.0, b1 = 0.0;
    for (int l = threadIdx.x; l < nloc; l += kResBlock) {
      sx[l] = fma(alpha, spp[l], sx[l]);
      const double ri = fma(-alpha, sq[l], sr[l]);
      const double zi = __ldg(dinv + r0 + l) * ri;
      sr[l] = ri;
      sz[l] = zi;
      zg[r0 + l] = zi;
      b0 += ri * zi;
      b1 += ri * ri;
    }
    {
      double v[2] = {b0, b1};
      block_sum<2, kResBlock>(v, sred);
      if (threadIdx.x == 0) { partB[blockIdx.x] = v[0]; partB[nb + blockIdx.x] = v[1]; }
    }
    grid_barrier(bar, ++nbar * nb);  // new z visible to every CTA's gathers
    all_sum<2>(partB, nb, bcast, t2);
    rz_old = rz;
    rz = t2[0];
    rr = t2[1];
  }
  for (int l = threadIdx.x; l < nloc; l += kResBlock) x_out[r0 + l] = sx[l];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    red[AB_RED_RZN] = rz;
    red[AB_RED_RR] = rr;
    red[AB_RED_ITERS] = (double)it;
    sc[AB_SC_BB] = bb;
  }
}

// ---------------------------------------------------------------------------
// Resident CG, tensor-memory form (k_cg_tmem).  Same algorithm and local
// column map as k_cg_resident_local, organised for sm_100a:
//  * the per-row CG vectors x, r, p, q and D^-1 live in TENSOR MEMORY (256 KB
//    per SM, tcgen05.ld/st, no tensor-core use): each consumer warp owns the
//    rows of its slices in its 32-lane quarter of TMEM, so shared memory only
//    holds z (own rows + ghosts);
//  * one producer warp streams the CTA's SELL slices (values + 16-bit local
//    columns) into a shared-memory ring with bulk asynchronous copies
//    (cp.async.bulk -> UBLKCP, mbarrier full/empty handshake).  The matrix
//    does not change, so the producer runs ahead across the grid barriers:
//    the next iteration's first slices land while the reductions complete;
//  * kTmNC consumer warps gather z from shared memory and synchronise among
//    themselves with a named barrier; the producer never joins them.
// Slice sl of the CTA is consumed by warp sl % kTmNC (row slot sl / kTmNC).
// Iterates equal k_cg_resident_local's (same per-row operation order); the
// dot products are summed in a different (fixed) tree.
// ---------------------------------------------------------------------------
constexpr int kTmNC = 24;
constexpr int kTmThreads = (kTmNC + 1) * 32;
constexpr int kTmCols = (512 / (kTmNC / 4)) & ~1;  // TMEM columns per consumer warp
constexpr int kTmMaxSlots = kTmCols / 10;   // row slots per thread (5 doubles each)

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(kTmNC * 32) : "memory"); }

__device__ __forceinline__ void mb_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa32(b)) : "memory");
}
__device__ __forceinline__ bool mb_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(sa32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  while (!mb_test(b, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sa32(dst)),
               "l"(src), "r"(bytes), "r"(sa32(b))
               : "memory");
}



// Sum over the consumer warps (valid in warp 0); sm >= NV * kTmNC doubles.
template <int NV>
__device__ __forceinline__ void cons_sum(double (&v)[NV], double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sm[k * kTmNC + warp] = v[k];
  cbar();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = lane < kTmNC ? sm[k * kTmNC + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      v[k] = t;
    }
  }
}

__device__ __forceinline__ void cons_grid_barrier(unsigned* cnt, unsigned target) {
  cbar();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
    } while (v < target);
  }
  cbar();
}

// Ordered sum of nb per-CTA partials (nb <= kTmNC * 32), identical in every CTA.
template <int NV>
__device__ __forceinline__ void cons_all_sum(const double* part, int nb, double* sm, double* bcast,
                                             double (&out)[NV]) {
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = (int)threadIdx.x < nb ? __ldcg(part + (size_t)k * nb + threadIdx.x) : 0.0;
  cons_sum<NV>(v, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) bcast[k] = v[k];
  cbar();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = bcast[k];
}

struct TmLayout {
  int ring;      // slots
  int maxw;      // widest slice (entries per lane)
  int kslots;    // row slots per consumer thread
  int group;     // slices per chunk (one bulk copy)
};

__global__ void __launch_bounds__(kTmThreads, 1) k_cg_tmem(
    int64_t n, int64_t rows_per_cta, int max_ghost, TmLayout L, const int64_t* __restrict__ sp,
    const unsigned char* __restrict__ packed, const int32_t* __restrict__ gptr,
    const int32_t* __restrict__ gidx, const int32_t* __restrict__ perm, const double* __restrict__ b_in,
    double* b_zero, const uint8_t* __restrict__ fixed, const double* __restrict__ dinv, double* __restrict__ x_out,
    double* zg, int maxit, double tol, double* red, double* sc, double* part, unsigned* bar) {
  extern __shared__ __align__(128) unsigned char tsm[];
  __shared__ double sred[2 * kTmNC];
  __shared__ double bcast[4];
  __shared__ uint32_t s_taddr;
  __shared__ volatile int s_stop;  // iteration at which the consumers stopped (-1: running)
  __shared__ volatile int s_seq[64];  // chunk sequence number last issued into each slot
  const int nb = gridDim.x;
  const int64_t RB = rows_per_cta;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int64_t r1 = r0 + RB < n ? r0 + RB : n;
  const int nloc = r1 > r0 ? (int)(r1 - r0) : 0;
  const int nsl = (nloc + 31) >> 5;
  const int64_t s_first = r0 >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g0 = gptr[blockIdx.x];
  const int ng = gptr[blockIdx.x + 1] - g0;
  const int G = L.group;
  const int nch = (nsl + G - 1) / G;  // chunks per iteration
  const uint32_t slot_bytes = (uint32_t)(G * L.maxw) * 320u;
  // shared memory carve-up
  double* sz = reinterpret_cast<double*>(tsm);                     // [RB + max_ghost]
  size_t off = ((size_t)(RB + max_ghost) * 8 + 127) & ~(size_t)127;
  unsigned char* ring = tsm + off;                                 // [ring][slot_bytes]
  off += (size_t)L.ring * slot_bytes;
  int64_t* ssp = reinterpret_cast<int64_t*>(tsm + off);            // [nsl + 1]
  off += ((size_t)(RB / 32 + 1) * 8 + 15) & ~(size_t)15;
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + off);          // [ring]
  uint64_t* empty = full + L.ring;                                  // [ring]
  off += (size_t)2 * L.ring * 8;
  int32_t* sgid = reinterpret_cast<int32_t*>(tsm + off);           // [max_ghost]

  for (int k = threadIdx.x; k <= nsl; k += kTmThreads) ssp[k] = sp[s_first + k];
  for (int k = threadIdx.x; k < ng; k += kTmThreads) sgid[k] = gidx[g0 + k];
  if (threadIdx.x == 0) {
    for (int k = 0; k < L.ring; ++k) {
      mb_init(full + k, 1);
      mb_init(empty + k, (unsigned)G);
      s_seq[k] = -1;
    }
    s_stop = -1;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa32(&s_taddr))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  if (warp == kTmNC) {
    // ================= producer: stream the slices, iteration after iteration
    if (lane == 0) {
      // chunk Q = it * nch + c covers slices [cG, min(cG + G, nsl)): one bulk
      // copy of their packed values + columns (10 bytes per entry, contiguous
      // in the packed buffer).  Counters kept incrementally (no division).
      const int total = maxit * nch;
      int q = 0, it = 0, c = 0, slot = 0;
      uint32_t par = 0;
      for (; q < total; ++q) {
        bool stop = false;
        if (q >= L.ring) {
          while (!mb_test(empty + slot, par ^ 1u)) {
            const int st = s_stop;
            if (st >= 0 && it >= st) { stop = true; break; }
          }
        }
        if (!stop) {
          const int st = s_stop;
          if (st >= 0 && it >= st) stop = true;
        }
        if (stop) break;
        const int c0 = c * G, c1 = c0 + G < nsl ? c0 + G : nsl;
        const int64_t e0 = ssp[c0];
        const uint32_t bytes = (uint32_t)(ssp[c1] - e0) * 10u;
        mb_expect_tx(full + slot, bytes);
        bulk_g2s(ring + (size_t)slot * slot_bytes, packed + 10 * e0, bytes, full + slot);
        for (int k = c1 - c0; k < G; ++k) mb_arrive(empty + slot);  // slices a short chunk lacks
        s_seq[slot] = q;
        if (++slot == L.ring) { slot = 0; par ^= 1u; }
        if (++c == nch) { c = 0; ++it; }
      }
      // drain: copies issued but never consumed must land before exit
      const int st = s_stop;
      const int consumed = st >= 0 ? st * nch : total;
      for (int k = (consumed > q - L.ring ? consumed : q - L.ring); k < q; ++k)
        mb_wait(full + (k % L.ring), (uint32_t)((k / L.ring) & 1));
    }
    return;
  }

  // ================= consumers
  const uint32_t tbase = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kTmCols);
  const int K = L.kslots;
  auto tcol = [&](int v, int k) -> uint32_t { return tbase + (uint32_t)(v * 2 * K + 2 * k); };
  enum { VX = 0, VR = 1, VP = 2, VQ = 3, VD = 4 };
  double* partA = part;
  double* partB = part + nb;
  double* partI = part + 3 * (size_t)nb;
  unsigned nbar = 0;

  // init: r = b (fixed rows 0), z = D^-1 r, x = p = q = 0
  double a0 = 0.0, a1 = 0.0;
  for (int k = 0; k < K; ++k) {
    const int sl = warp + k * kTmNC;
    const int l = sl * 32 + lane;
    double ri = 0.0, di = 0.0;
    if (sl < nsl && l < nloc) {
      const int64_t i = r0 + l;
      const int64_t ni = perm ? (int64_t)perm[i] : i;
      ri = b_in[ni];
      if (fixed && fixed[i]) ri = 0.0;
      if (b_zero) b_zero[ni] = 0.0;
      di = dinv[i];
      const double zi = di * ri;
      sz[l] = zi;
      zg[i] = zi;
      a0 += ri * zi;
      a1 += ri * ri;
    }
    tm_st(tcol(VX, k), 0.0);
    tm_st(tcol(VR, k), ri);
    tm_st(tcol(VP, k), 0.0);
    tm_st(tcol(VQ, k), 0.0);
    tm_st(tcol(VD, k), di);
  }
  tm_wait_st();
  {
    double v[2] = {a0, a1};
    cons_sum<2>(v, sred);
    if (threadIdx.x == 0) { partI[blockIdx.x] = v[0]; partI[nb + blockIdx.x] = v[1]; }
  }
  cons_grid_barrier(bar, ++nbar * nb);
  double t2[2];
  cons_all_sum<2>(partI, nb, sred, bcast, t2);
  double rz = t2[0], rr = t2[1];
  const double bb = rr;
  double rz_old = 0.0;
  int it = 0;
  for (; it < maxit; ++it) {
    if (tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) break;
    const double beta = rz_old != 0.0 ? rz / rz_old : 0.0;
    for (int k = threadIdx.x; k < ng; k += kTmNC * 32) sz[RB + k] = __ldcg(zg + sgid[k]);
    cbar();
    // ---- phase A
    double pq = 0.0;
    for (int k = 0; k < K; ++k) {
      const int sl = warp + k * kTmNC;
      if (sl >= nsl) break;  // warp-uniform
      uint32_t plo, phi, qlo, qhi;
      tm_ld(tcol(VP, k), plo, phi);
      tm_ld(tcol(VQ, k), qlo, qhi);
      const int c = sl / G;
      const int qi = it * nch + c;
      const unsigned qd = (unsigned)qi / (unsigned)L.ring;
      const int slot = (int)((unsigned)qi - qd * (unsigned)L.ring);
      while (s_seq[slot] != qi) {
      }
      mb_wait(full + slot, qd & 1u);
      const int64_t ce0 = ssp[c * G], ce1 = ssp[(c * G + G) < nsl ? c * G + G : nsl];
      const int64_t so = ssp[sl] - ce0;
      const double* sv = reinterpret_cast<const double*>(ring + (size_t)slot * slot_bytes) + so;
      const uint16_t* sc16 =
          reinterpret_cast<const uint16_t*>(ring + (size_t)slot * slot_bytes + (size_t)(ce1 - ce0) * 8) + so;
      const int width = (int)((ssp[sl + 1] - ssp[sl]) >> 5);
      double acc = 0.0;
      for (int j0 = 0; j0 < width; j0 += 8) {
        unsigned cj[8];
        double aj[8], gj[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool ok = j0 + u < width;
          cj[u] = ok ? (unsigned)sc16[(j0 + u) * 32 + lane] : 0u;
          aj[u] = ok ? sv[(j0 + u) * 32 + lane] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) gj[u] = sz[cj[u]];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(aj[u], gj[u], acc);
      }
      __syncwarp();
      if (lane == 0) mb_arrive(empty + slot);
      tm_wait_ld();
      const int l = sl * 32 + lane;
      const double p = fma(beta, tm_val(plo, phi), l < nloc ? sz[l] : 0.0);
      const double q = fma(beta, tm_val(qlo, qhi), acc);
      tm_st(tcol(VP, k), p);
      tm_st(tcol(VQ, k), q);
      if (l < nloc) pq += p * q;
    }
    tm_wait_st();
    {
      double v[1] = {pq};
      cons_sum<1>(v, sred);
      if (threadIdx.x == 0) partA[blockIdx.x] = v[0];
    }
    cons_grid_barrier(bar, ++nbar * nb);
    double t1[1];
    cons_all_sum<1>(partA, nb, sred, bcast, t1);
    const double alpha = t1[0] != 0.0 ? rz / t1[0] : 0.0;
    // ---- phase B: x += alpha p, r -= alpha q, z = D^-1 r
    double b0 = 0.0, b1 = 0.0;
    for (int k = 0; k < K; ++k) {
      const int sl = warp + k * kTmNC;
      if (sl >= nsl) break;
      uint32_t v[5][2];
      tm_ld(tcol(VX, k), v[0][0], v[0][1]);
      tm_ld(tcol(VR, k), v[1][0], v[1][1]);
      tm_ld(tcol(VP, k), v[2][0], v[2][1]);
      tm_ld(tcol(VQ, k), v[3][0], v[3][1]);
      tm_ld(tcol(VD, k), v[4][0], v[4][1]);
      tm_wait_ld();
      const double xi = fma(alpha, tm_val(v[2][0], v[2][1]), tm_val(v[0][0], v[0][1]));
      const double ri = fma(-alpha, tm_val(v[3][0], v[3][1]), tm_val(v[1][0], v[1][1]));
      const double zi = tm_val(v[4][0], v[4][1]) * ri;
      tm_st(tcol(VX, k), xi);
      tm_st(tcol(VR, k), ri);
      const int l = sl * 32 + lane;
      if (l < nloc) {
        sz[l] = zi;
        zg[r0 + l] = zi;
        b0 += ri * zi;
        b1 += ri * ri;
      }
    }
    tm_wait_st();
    {
      double v[2] = {b0, b1};
      cons_sum<2>(v, sred);
      if (threadIdx.x == 0) { partB[blockIdx.x] = v[0]; partB[nb + blockIdx.x] = v[1]; }
    }
    cons_grid_barrier(bar, ++nbar * nb);
    cons_all_sum<2>(partB, nb, sred, bcast, t2);
    rz_old = rz;
    rz = t2[0];
    rr = t2[1];
  }
  if (threadIdx.x == 0) s_stop = it;
  // x -> node order
  for (int k = 0; k < K; ++k) {
    const int sl = warp + k * kTmNC;
    if (sl >= nsl) break;
    uint32_t lo, hi;
    tm_ld(tcol(VX, k), lo, hi);
    tm_wait_ld();
    const int l = sl * 32 + lane;
    if (l < nloc) x_out[perm ? (int64_t)perm[r0 + l] : r0 + l] = tm_val(lo, hi);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cbar();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_taddr) : "memory");
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    red[AB_RED_RZN] = rz;
    red[AB_RED_RR] = rr;
    red[AB_RED_ITERS] = (double)it;
    sc[AB_SC_BB] = bb;
  }
}

// ---------------------------------------------------------------------------
// Single-reduction resident CG (Chronopoulos-Gear form, k_cg_cg1).  Same
// preconditioned CG in exact arithmetic, reorganised so that each iteration
// has ONE grid-wide reduction:
//   s = A z (SpMV on z); gamma = r.z, delta = z.s, rr = r.r  -> one reduction
//   beta = gamma / gamma_old;  alpha = gamma / (delta - beta gamma / alpha_old)
//   p = z + beta p;  q = s + beta q (= A p);  x += alpha p;  r -= alpha q;
//   z = D^-1 r  -> published to the neighbouring CTAs by per-CTA epoch flags
// The second grid barrier of the two-reduction form becomes a wait on the
// CTAs that own this CTA's ghost rows (z visibility is the only thing the
// next SpMV needs); the grid barrier of the reduction follows every SpMV, so
// no CTA can overwrite z while a neighbour still gathers it.  x and s = A z
// wait in tensor memory (columns 0-15 / 16-31 of the thread's lane), r, p,
// q, z + ghosts stay in shared memory.  Row mapping everywhere: slice sl =
// warp + 32 k, lane = row in the slice.
// ---------------------------------------------------------------------------
constexpr int kCg1Rounds = 8;  // slices per warp: rows_per_cta <= 8 * 1024

__global__ void __launch_bounds__(kResBlock, 1) k_cg_cg1(
    int64_t n, int64_t rows_per_cta, int max_ghost, const int64_t* __restrict__ sp,
    const uint16_t* __restrict__ lcol, const double* __restrict__ sval, const int32_t* __restrict__ gptr,
    const int32_t* __restrict__ gidx, const int32_t* __restrict__ nbr_ptr, const int32_t* __restrict__ nbr,
    const int32_t* __restrict__ perm, const double* __restrict__ b_in, double* b_zero,
    const uint8_t* __restrict__ fixed, const double* __restrict__ dinv, double* __restrict__ x_out, double* zg,
    int maxit, double tol, double* red, double* sc, double* part, unsigned* bar, unsigned* flags) {
  extern __shared__ double smem[];
  __shared__ double sred[3 * (kResBlock / 32)];
  __shared__ double bcast[4];
  __shared__ uint32_t s_taddr;
  const int nb = gridDim.x;
  const int64_t RB = rows_per_cta;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int64_t r1 = r0 + RB < n ? r0 + RB : n;
  const int nloc = r1 > r0 ? (int)(r1 - r0) : 0;
  double* sr = smem;
  double* spp = sr + RB;
  double* sq = spp + RB;
  double* sz = sq + RB;  // [RB] own rows, then [max_ghost] ghosts
  int64_t* tsp = reinterpret_cast<int64_t*>(sz + RB + max_ghost);
  int32_t* tg = reinterpret_cast<int32_t*>(tsp + RB / 32 + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsl = (nloc + 31) >> 5;
  const int64_t s_first = r0 >> 5;
  const int g0 = gptr[blockIdx.x];
  const int ng = gptr[blockIdx.x + 1] - g0;
  const int nb0 = nbr_ptr[blockIdx.x], nnb = nbr_ptr[blockIdx.x + 1] - nb0;
  for (int k = threadIdx.x; k <= nsl; k += kResBlock) tsp[k] = sp[s_first + k];
  for (int k = threadIdx.x; k < ng; k += kResBlock) tg[k] = gidx[g0 + k];
  const uint32_t taddr = tmem_alloc_all(&s_taddr);  // includes __syncthreads
  const uint32_t tx = taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
  unsigned nbar = 0;

  // ---- init: r = b (fixed rows 0), z = D^-1 r, x = p = q = 0
#pragma unroll
  for (int k = 0; k < kCg1Rounds; ++k) {
    const int sl = warp + k * (kResBlock / 32);
    const int l = sl * 32 + lane;
    if (sl < nsl && l < nloc) {
      const int64_t i = r0 + l;
      const int64_t ni = perm ? (int64_t)perm[i] : i;
      double ri = b_in[ni];
      if (fixed && fixed[i]) ri = 0.0;
      if (b_zero) b_zero[ni] = 0.0;
      const double zi = dinv[i] * ri;
      sr[l] = ri; sz[l] = zi; spp[l] = 0.0; sq[l] = 0.0;
      zg[i] = zi;
    }
    tm_st(tx + 2 * k, 0.0);
  }
  tm_wait_st();
  grid_barrier(bar, ++nbar * nb);  // z visible to every CTA

  double gamma_old = 0.0, alpha_old = 0.0, bb = 0.0, gamma = 0.0, rr = 0.0;
  int it = 0;
  bool converged = false;
  for (; it < maxit; ++it) {
    // ---- ghost z -> shared memory
    for (int k = threadIdx.x; k < ng; k += kResBlock) sz[RB + k] = __ldcg(zg + tg[k]);
    __syncthreads();
    // ---- s = A z -> TMEM; local gamma = r.z, delta = z.s, rr = r.r
    double dg = 0.0, dd = 0.0, dr = 0.0;
#pragma unroll 1
    for (int k = 0; k * (kResBlock / 32) + warp < nsl; ++k) {
      const int sl = warp + k * (kResBlock / 32);
      const double az = sell_row_dot_smem<kLocChunk>(tsp, lcol, sval, sz, sl, lane);
      tm_st(tx + 16 + 2 * k, az);
      const int l = sl * 32 + lane;
      if (l < nloc) {
        const double zi = sz[l], ri = sr[l];
        dg += ri * zi;
        dd += zi * az;
        dr += ri * ri;
      }
    }
    // D^-1 of this thread's rows: in flight across the reduction
    double dv[kCg1Rounds];
#pragma unroll
    for (int k = 0; k < kCg1Rounds; ++k) {
      const int l = (warp + k * (kResBlock / 32)) * 32 + lane;
      dv[k] = l < nloc ? __ldg(dinv + r0 + l) : 0.0;
    }
    double t3[3];
    {
      double v[3] = {dg, dd, dr};
      block_sum<3, kResBlock>(v, sred);
      if (threadIdx.x == 0) {
        part[blockIdx.x] = v[0];
        part[nb + blockIdx.x] = v[1];
        part[2 * nb + blockIdx.x] = v[2];
      }
      grid_barrier(bar, ++nbar * nb);
      all_sum_par<3>(part, nb, sred, bcast, t3);
    }
    gamma = t3[0];
    rr = t3[2];
    if (it == 0) bb = rr;
    if (tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) {
      converged = true;
      break;
    }
    const double delta = t3[1];
    double alpha, beta;
    if (it == 0) {
      beta = 0.0;
      alpha = delta != 0.0 ? gamma / delta : 0.0;
    } else {
      beta = gamma_old != 0.0 ? gamma / gamma_old : 0.0;
      const double den = delta - (alpha_old != 0.0 ? beta * gamma / alpha_old : 0.0);
      alpha = den != 0.0 ? gamma / den : 0.0;
    }
    // ---- p = z + beta p, q = s + beta q, x += alpha p, r -= alpha q, z = D^-1 r
    tm_wait_st();
#pragma unroll
    for (int k = 0; k < kCg1Rounds; ++k) {
      const int sl = warp + k * (kResBlock / 32);
      if (sl >= nsl) break;  // warp-uniform
      uint32_t xl, xh, sl32, sh;
      tm_ld(tx + 2 * k, xl, xh);
      tm_ld(tx + 16 + 2 * k, sl32, sh);
      tm_wait_ld();
      const double xo = tm_val(xl, xh), si = tm_val(sl32, sh);
      const int l = sl * 32 + lane;
      double xn = xo;
      if (l < nloc) {
        const double p = fma(beta, spp[l], sz[l]);
        const double q = fma(beta, sq[l], si);
        xn = fma(alpha, p, xo);
        const double ri = fma(-alpha, q, sr[l]);
        const double zi = dv[k] * ri;
        spp[l] = p;
        sq[l] = q;
        sr[l] = ri;
        sz[l] = zi;
        zg[r0 + l] = zi;
      }
      tm_st(tx + 2 * k, xn);
    }
    gamma_old = gamma;
    alpha_old = alpha;
    // ---- publish z; wait for the CTAs owning this CTA's ghost rows
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"((unsigned)(it + 1))
                   : "memory");
    if ((int)threadIdx.x < nnb) {
      const unsigned* f = flags + nbr[nb0 + threadIdx.x];
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      } while (v < (unsigned)(it + 1));
    }
    __syncthreads();
  }
  if (!converged) {  // residual of the final iterate (one more reduction)
    double v[2] = {0.0, 0.0};
    for (int l = threadIdx.x; l < nloc; l += kResBlock) {
      v[0] += sr[l] * sz[l];
      v[1] += sr[l] * sr[l];
    }
    block_sum<2, kResBlock>(v, sred);
    if (threadIdx.x == 0) {
      part[blockIdx.x] = v[0];
      part[nb + blockIdx.x] = v[1];
    }
    grid_barrier(bar, ++nbar * nb);
    double t2[2];
    all_sum_par<2>(part, nb, sred, bcast, t2);
    gamma = t2[0];
    rr = t2[1];
    if (maxit == 0) bb = rr;
  }
  tm_wait_st();
#pragma unroll
  for (int k = 0; k < kCg1Rounds; ++k) {
    const int sl = warp + k * (kResBlock / 32);
    uint32_t lo, hi;
    tm_ld(tx + 2 * k, lo, hi);
    tm_wait_ld();
    const int l = sl * 32 + lane;
    if (sl < nsl && l < nloc) x_out[perm ? (int64_t)perm[r0 + l] : r0 + l] = tm_val(lo, hi);
  }
  tmem_free_all(taddr);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    red[AB_RED_RZN] = gamma;
    red[AB_RED_RR] = rr;
    red[AB_RED_ITERS] = (double)it;
    sc[AB_SC_BB] = bb;
  }
}
