// Single-barrier variant of k_pipe: four metadata stages and
// two slot buffers let the window-node reductions of block i-1 (phase D) and
// the elements of block i (phase C) run back to back in every thread, so a
// CTA meets one barrier per block and warps that finish D early go straight
// on to C.  Iteration i:
//   wait own gathers(i); barrier X (gathers(i) visible, C(i-1) and D(i-2) done)
//   thread 0: bulk metadata(i+2) -> stage (i+2)%4 (last read by D(i-2))
//   wait metadata(i+1); cp.async gathers(i+1) -> nodes[(i+1)&1] (read by C(i-1))
//   D(i-1) from slots[(i-1)&1];  C(i) -> slots[i&1] (last read by D(i-2))
template <int NN, int NV, int BLOCK>
struct Pipe1Smem {
  using L = PipeSmem<NN, NV, BLOCK>;
  static __host__ __device__ size_t total(int wmax) {
    return 4 * L::meta_bytes(wmax) + 2 * L::node_bytes(wmax) + 2 * L::slot_bytes();
  }
};

#ifndef PIPE1_OCC_K2
#define PIPE1_OCC_K2 4
#endif
template <int R, int OP> struct Pipe1Occ { static constexpr int value = 1; };
template <> struct Pipe1Occ<AB_RULE_TET4, OP_MOMENTUM> { static constexpr int value = PIPE1_OCC_K2; };

template <int R, int OP, int BLOCK>
__global__ void __launch_bounds__(BLOCK, Pipe1Occ<R, OP>::value) k_pipe1(CatP c, WinP w, ab_phys ph, double scale,
                                                                         const double* __restrict__ f,
                                                                         double* __restrict__ out, int64_t n_blocks) {
  constexpr int NN = RuleT<R>::NN;
  constexpr int NV = OpT<R, OP>::NV, NC = OpT<R, OP>::NC, STRIDE = OpT<R, OP>::STRIDE;
  using L = PipeSmem<NN, NV, BLOCK>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[4];
  const int wmax = w.wmax;
  double* nodes0 = reinterpret_cast<double*>(smem + 4 * L::meta_bytes(wmax));
  double* slots0 = reinterpret_cast<double*>(smem + 4 * L::meta_bytes(wmax) + 2 * L::node_bytes(wmax));
  const int64_t stride = gridDim.x;
  const int64_t b_first = blockIdx.x;
  if (b_first >= n_blocks) return;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) mbar_init1(&bars[q]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // descriptors of blocks i-1, i, i+1, i+2 (dp, d0, d1, d2)
  int4 d0 = __ldg(w.desc + b_first);
  int4 d1 = b_first + stride < n_blocks ? __ldg(w.desc + b_first + stride) : d0;
  int4 d2 = b_first + 2 * stride < n_blocks ? __ldg(w.desc + b_first + 2 * stride) : d0;
  int4 dp = d0;
  if (threadIdx.x == 0) {
    issue_meta<NN>(w, c.n, b_first, d0, meta_ptr<NN, NV, BLOCK>(smem, wmax, 0), &bars[0]);
    if (b_first + stride < n_blocks)
      issue_meta<NN>(w, c.n, b_first + stride, d1, meta_ptr<NN, NV, BLOCK>(smem, wmax, 1), &bars[1]);
  }
  mbar_wait_parity(&bars[0], 0);
  issue_nodes<NV, BLOCK>(c, f, wmax, meta_ptr<NN, NV, BLOCK>(smem, wmax, 0), block_view(w, d0), nodes0);

  // D: ordered per-window-node sums of block `it` (stage it%4, slots it&1)
  auto phase_d = [&](int it_d, const int4& dd) {
    const MetaPtr md = meta_ptr<NN, NV, BLOCK>(smem, wmax, it_d & 3);
    const BlockView vd = block_view(w, dd);
    const double* slots = slots0 + (size_t)(it_d & 1) * 3 * NN * BLOCK;
    for (int k = threadIdx.x; k < vd.nw; k += BLOCK) {
      const int node = md.wnode[vd.skip_wnode + k];
      const int s0 = md.wptr[vd.skip_wptr + k] - vd.s_lo, s1 = md.wptr[vd.skip_wptr + k + 1] - vd.s_lo;
      double acc[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) acc[q] = 0.0;
      for (int t0 = s0; t0 < s1; t0 += 8) {
        int sl[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) sl[u] = t0 + u < s1 ? (int)md.wslot[vd.skip_wslot + t0 + u] : -1;
        double vq[8][NC];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int slot = sl[u] < 0 ? 0 : sl[u];
          const int a = slot % NN, el = slot / NN;
#pragma unroll
          for (int q = 0; q < NC; ++q) vq[u][q] = slots[(q * NN + a) * BLOCK + el];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (sl[u] >= 0)
#pragma unroll
            for (int q = 0; q < NC; ++q) acc[q] += vq[u][q];
      }
#pragma unroll
      for (int q = 0; q < NC; ++q) red_add(out + (int64_t)node * STRIDE + q, acc[q]);
    }
  };

  int it = 0;
  for (int64_t b = b_first; b < n_blocks; b += stride, ++it) {
    double* nodes_cur = nodes0 + (size_t)(it & 1) * NV * wmax;
    double* nodes_nxt = nodes0 + (size_t)((it + 1) & 1) * NV * wmax;
    double* slots = slots0 + (size_t)(it & 1) * 3 * NN * BLOCK;
    const int64_t b2 = b + 2 * stride, b3 = b + 3 * stride;
    const int4 d3 = b3 < n_blocks ? __ldg(w.desc + b3) : d0;
    cp_async_wait<0>();
    __syncthreads();  // X
    if (threadIdx.x == 0 && b2 < n_blocks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_meta<NN>(w, c.n, b2, d2, meta_ptr<NN, NV, BLOCK>(smem, wmax, (it + 2) & 3), &bars[(it + 2) & 3]);
    }
    if (b + stride < n_blocks) {
      mbar_wait_parity(&bars[(it + 1) & 3], (uint32_t)(((it + 1) >> 2) & 1));
      issue_nodes<NV, BLOCK>(c, f, wmax, meta_ptr<NN, NV, BLOCK>(smem, wmax, (it + 1) & 3), block_view(w, d1),
                             nodes_nxt);
    }
    if (it > 0) phase_d(it - 1, dp);
    // C: elements of this block
    const MetaPtr mc = meta_ptr<NN, NV, BLOCK>(smem, wmax, it & 3);
    const int64_t e = b * BLOCK + threadIdx.x;
    if (e < c.n) {
      double x[NN][3], fv[NN][NV == 6 ? 3 : 1];
      int li[NN];
      if constexpr (NN == 4) {
        const uint2 lv = *reinterpret_cast<const uint2*>(mc.loc + threadIdx.x * NN);
        li[0] = lv.x & 0xffff; li[1] = lv.x >> 16; li[2] = lv.y & 0xffff; li[3] = lv.y >> 16;
      } else {
#pragma unroll
        for (int a = 0; a < NN; ++a) li[a] = mc.loc[threadIdx.x * NN + a];
      }
      const double2* pr = reinterpret_cast<const double2*>(nodes_cur);
#pragma unroll
      for (int a = 0; a < NN; ++a) {
        const int l = li[a];
        const double2 xy = pr[l], zf = pr[wmax + l];
        x[a][0] = xy.x;
        x[a][1] = xy.y;
        x[a][2] = zf.x;
        fv[a][0] = zf.y;
        if constexpr (NV == 6) {
          const double2 vw = pr[2 * wmax + l];
          fv[a][1] = vw.x;
          fv[a][2] = vw.y;
        }
      }
      unwrap<NN>(c, x);
      if constexpr (OP == OP_MOMENTUM) {
        momentum_element<R, NN>(ph, x, fv, [&](int a, const double (&v)[3]) {
#pragma unroll
          for (int k = 0; k < 3; ++k) slots[(k * NN + a) * BLOCK + threadIdx.x] = v[k];
        });
      } else {
        double r[NN][NC];
#pragma unroll
        for (int a = 0; a < NN; ++a)
#pragma unroll
          for (int k = 0; k < NC; ++k) r[a][k] = 0.0;
        if constexpr (OP == OP_DIVERGENCE) divergence_element<R, NN>(scale, x, fv, r);
        if constexpr (OP == OP_GRADIENT) gradient_element<R, NN>(scale, x, fv, r);
#pragma unroll
        for (int a = 0; a < NN; ++a)
#pragma unroll
          for (int k = 0; k < NC; ++k) slots[(k * NN + a) * BLOCK + threadIdx.x] = r[a][k];
      }
    } else {
#pragma unroll
      for (int a = 0; a < NN; ++a)
#pragma unroll
        for (int k = 0; k < NC; ++k) slots[(k * NN + a) * BLOCK + threadIdx.x] = 0.0;
    }
    dp = d0;
    d0 = d1;
    d1 = d2;
    d2 = d3;
  }
  __syncthreads();
  phase_d(it - 1, dp);
}

template <int R, int OP, int BLOCK>
static int launch_pipe1(const CatP& c, const WinP& w, const ab_phys& ph, double scale, const double* f, double* out,
                        cudaStream_t stream) {
  constexpr int NN = RuleT<R>::NN;
  constexpr int NV = OpT<R, OP>::NV;
  const size_t smem = Pipe1Smem<NN, NV, BLOCK>::total(w.wmax);
  auto kern = k_pipe1<R, OP, BLOCK>;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail("single-barrier element kernel: shared memory request rejected");
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLOCK, smem);
  if (per_sm < 1) return fail("single-barrier element kernel does not fit on an SM");
  const int64_t n_blocks = (c.n + BLOCK - 1) / BLOCK;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > n_blocks) grid = n_blocks;
  kern<<<(unsigned)grid, BLOCK, smem, stream>>>(c, w, ph, scale, f, out, n_blocks);
  return check_launch("k_pipe1");
}

