// Rejected variant (round 2; measured slower and superseded by the tiled
// 16-bit columns of ab_cg_spmv_tile; not built).  Column-compressed SELL-32
// for the two-kernel CG: per slice 16-bit column offsets from cbase[s] when
// the slice's columns span < 65536 rows, int32 otherwise.  On the C3 system
// it cut the SpMV's DRAM bytes 9% but ran 207-210 us like the int32 form
// (the per-entry z gather sets the pace; profiles/r2_spmv_c3_lab.md).  To
// rebuild: paste the device helpers into ab_cg_common.cuh, the kernels and
// entry points into ab_solver.cu, the declarations into include/alyab200.h.

/* Column-compressed SELL-32 for the single-domain two-kernel CG: the same
 * slices, values and entry order as an ab_sell; slice s keeps its columns
 * as uint16 offsets from cbase[s] when they span < 65536 rows (int32 and
 * cbase[s] = -1 otherwise), at byte offset cptr[s] of `cols` (16-byte
 * aligned).  In the Hilbert row order most slices qualify, which cuts the
 * column stream - a third of the matrix bytes - nearly in half.
 * ab_sell16_plan: cbase and per-slice byte counts from an ab_sell; the
 * caller scans the counts into cptr; ab_sell16_fill writes the columns.
 * ab_cg_spmv16 = ab_cg_spmv(with_dot = 1, own = NULL), bitwise the same. */
typedef struct ab_sell16 {
  int64_t n_rows;
  int64_t n_slices;
  const int64_t* slice_ptr;
  const int64_t* cptr;
  const int32_t* cbase;
  const unsigned char* cols;
  const double* vals;
} ab_sell16;
int ab_sell16_plan(const ab_sell* a, int32_t* cbase, int64_t* bytes, void* stream);
int ab_sell16_fill(const ab_sell* a, const int32_t* cbase, const int64_t* cptr, unsigned char* cols, void* stream);
int ab_cg_spmv16(const ab_sell16* a, const double* z, double* p, double* q, double* red, double* sc, double* part,
                 uint32_t* cnt, void* stream);

// The same row product on the column-compressed SELL (ab_sell16): slice s
// stores its columns as 16-bit offsets from cbase[s] when they span < 64k
// rows, else as int32 (cbase[s] = -1); the branch is uniform per warp (one
// slice = one warp) and the FMA order is sell_row_dot's, so the result is
// bitwise the same.
#ifndef SPMV16_CHUNK
#define SPMV16_CHUNK 16
#endif
template <bool NEAR>
__device__ __forceinline__ double sell16_row_body(const unsigned char* __restrict__ cb, int64_t cofs, int cbase,
                                                  const double* __restrict__ sval, int64_t base, int lane, int width,
                                                  const double* zv) {
  constexpr int CH = SPMV16_CHUNK;
  double acc = 0.0;
  for (int j0 = 0; j0 < width; j0 += CH) {
    int c[CH];
    double a[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const bool ok = j0 + u < width;
      const int64_t k = (int64_t)(j0 + u) * 32 + lane;
      if constexpr (NEAR)
        c[u] = ok ? cbase + (int)__ldcs(reinterpret_cast<const uint16_t*>(cb + cofs) + k) : 0;
      else
        c[u] = ok ? __ldcs(reinterpret_cast<const int32_t*>(cb + cofs) + k) : 0;
      a[u] = ok ? __ldcs(sval + base + (int64_t)(j0 + u) * 32) : 0.0;
    }
    double g[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) g[u] = zv[c[u]];
#pragma unroll
    for (int u = 0; u < CH; ++u) acc = fma(a[u], g[u], acc);
  }
  return acc;
}

__device__ __forceinline__ double sell16_row_dot(const int64_t* __restrict__ sp, const int64_t* __restrict__ cptr,
                                                 const int32_t* __restrict__ cbase, const unsigned char* __restrict__ cb,
                                                 const double* __restrict__ sval, const double* zv, int64_t i) {
  const int64_t s = i >> 5;
  const int lane = (int)(i & 31);
  const int64_t base = sp[s] + lane;
  const int width = (int)((sp[s + 1] - sp[s]) >> 5);
  const int b = cbase[s];
  if (b >= 0) return sell16_row_body<true>(cb, cptr[s], b, sval, base, lane, width, zv);
  return sell16_row_body<false>(cb, cptr[s], 0, sval, base, lane, width, zv);
}

// Single domain on the column-compressed SELL (ab_sell16): the DOT form of
// k_cg_spmv with 2-byte columns in the slices that allow them.
#ifndef SPMV16_MINB
#define SPMV16_MINB 8  // 32 registers, full occupancy (1 block: 90 registers, 2x slower)
#endif
__global__ void __launch_bounds__(kCgBlock, SPMV16_MINB) k_cg_spmv16(int64_t n, const int64_t* __restrict__ sp,
                                                        const int64_t* __restrict__ cptr,
                                                        const int32_t* __restrict__ cbase,
                                                        const unsigned char* __restrict__ cb,
                                                        const double* __restrict__ sval, const double* __restrict__ z,
                                                        double* __restrict__ p, double* __restrict__ q, double* red,
                                                        double* sc, double* part, uint32_t* cnt) {
  const int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x;
  const double rz_old = sc[AB_SC_RZ];
  const double rz_new = red[AB_RED_RZN];
  const double beta = rz_old != 0.0 ? rz_new / rz_old : 0.0;
  double v[1] = {0.0};
  if (i < n) {
    const double az = sell16_row_dot(sp, cptr, cbase, cb, sval, z, i);
    const double pi = fma(beta, p[i], z[i]);
    const double qi = fma(beta, q[i], az);
    p[i] = pi;
    q[i] = qi;
    v[0] = pi * qi;
  }
  double tot[1];
  if (grid_sum<1, kCgBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
    red[AB_RED_PQ] = tot[0];
    sc[AB_SC_RZ] = rz_new;
  }
}

// Column span of every SELL slice (one warp per slice): cbase = min column
// if max - min < 65536, else -1; bytes = the slice's column bytes, 16-byte
// aligned (2 or 4 per stored entry).
__global__ void k_sell16_plan(int64_t ns, const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
                              int32_t* __restrict__ cbase, int64_t* __restrict__ bytes) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= ns) return;
  int lo = 0x7fffffff, hi = -1;
  for (int64_t k = sp[s] + lane; k < sp[s + 1]; k += 32) {
    const int c = scol[k];
    lo = min(lo, c);
    hi = max(hi, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) {
    const int64_t e = sp[s + 1] - sp[s];
    const bool near = hi < 0 || (int64_t)hi - lo < 65536;
    cbase[s] = near ? (hi < 0 ? 0 : lo) : -1;
    bytes[s] = ((near ? 2 : 4) * e + 15) / 16 * 16;
  }
}

__global__ void k_sell16_fill(int64_t ns, const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
                              const int32_t* __restrict__ cbase, const int64_t* __restrict__ cptr,
                              unsigned char* __restrict__ cb) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= ns) return;
  const int b = cbase[s];
  for (int64_t k = sp[s] + lane; k < sp[s + 1]; k += 32) {
    const int64_t j = k - sp[s];
    if (b >= 0)
      reinterpret_cast<uint16_t*>(cb + cptr[s])[j] = (uint16_t)(scol[k] - b);
    else
      reinterpret_cast<int32_t*>(cb + cptr[s])[j] = scol[k];
  }
}

int ab_sell16_plan(const ab_sell* a, int32_t* cbase, int64_t* bytes, void* stream) {
  if (!a || !cbase || !bytes) return fail("ab_sell16_plan: null argument");
  if (a->n_slices > 0)
    k_sell16_plan<<<grid_for(a->n_slices * 32, 256), 256, 0, S(stream)>>>(a->n_slices, a->slice_ptr, a->cols, cbase,
                                                                          bytes);
  return check_launch("ab_sell16_plan");
}

int ab_sell16_fill(const ab_sell* a, const int32_t* cbase, const int64_t* cptr, unsigned char* cols, void* stream) {
  if (!a || !cbase || !cptr || !cols) return fail("ab_sell16_fill: null argument");
  if (a->n_slices > 0)
    k_sell16_fill<<<grid_for(a->n_slices * 32, 256), 256, 0, S(stream)>>>(a->n_slices, a->slice_ptr, a->cols, cbase,
                                                                          cptr, cols);
  return check_launch("ab_sell16_fill");
}

int ab_cg_spmv16(const ab_sell16* a, const double* z, double* p, double* q, double* red, double* sc, double* part,
                 uint32_t* cnt, void* stream) {
  if (!a || !a->slice_ptr || !a->cptr || !a->cbase || !a->cols) return fail("ab_cg_spmv16: incomplete matrix");
  const int64_t n = a->n_rows;
  k_cg_spmv16<<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, a->slice_ptr, a->cptr, a->cbase, a->cols, a->vals,
                                                                 z, p, q, red, sc, part, cnt);
  return check_launch("ab_cg_spmv16");
}
