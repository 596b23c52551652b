// ---------------------------------------------------------------------------
// Warp-window element kernel (K2).  Every warp is an independent worker over
// 32-element blocks (SFC order) with its own node window: no CTA barrier
// anywhere, only __syncwarp.  Per block the builder (device.py,
// build_warp_windows) stores fixed-size records so a lane can prefetch its
// share with plain coalesced loads one or two blocks ahead:
//   loc  u16 [32][NN]   window index of each element node (element side)
//   perm u16 [32*NN]    element-node references sorted by window node, as the
//                       shared-memory slot offset a*32 + e; lane l owns
//                       sorted positions l*NN .. l*NN+NN-1
//   head u8  [32]       bit k of lane l: position l*NN+k starts a window node
//   wnode i32 [wcap]    window node ids (ascending; padding = n_nodes)
// Connectivity is padded to whole blocks with a virtual node n_nodes, so the
// last block needs no special case (its virtual node is never gathered and
// never reduced).  Phase D is a warp-wide segmented sum over the sorted
// references (fixed NN positions per lane + shuffle scan) followed by one
// fp64 reduction per window node and component: balanced across lanes.
// ---------------------------------------------------------------------------
struct WarpWinP {
  const uint16_t* __restrict__ loc;
  const uint16_t* __restrict__ perm;
  const uint8_t* __restrict__ head;
  const int32_t* __restrict__ wnode;
  int64_t n_blocks;
  int wcap;
  int n_nodes;
};

template <int NN>
struct LaneRec {
  uint16_t loc[NN], perm[NN];
  uint32_t head;
};

template <int NN>
__device__ __forceinline__ void load_rec(const WarpWinP& w, int64_t b, int lane, LaneRec<NN>& r) {
  const int64_t o = (b * 32 + lane) * NN;
  if constexpr (NN == 4) {
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(w.loc + o));
    const uint2 p = __ldg(reinterpret_cast<const uint2*>(w.perm + o));
    r.loc[0] = a.x & 0xffff; r.loc[1] = a.x >> 16; r.loc[2] = a.y & 0xffff; r.loc[3] = a.y >> 16;
    r.perm[0] = p.x & 0xffff; r.perm[1] = p.x >> 16; r.perm[2] = p.y & 0xffff; r.perm[3] = p.y >> 16;
  } else {
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      r.loc[a] = __ldg(w.loc + o + a);
      r.perm[a] = __ldg(w.perm + o + a);
    }
  }
  r.head = __ldg(w.head + b * 32 + lane);
}

template <int WK>
__device__ __forceinline__ void load_wn(const WarpWinP& w, int64_t b, int lane, int (&wn)[WK]) {
#pragma unroll
  for (int t = 0; t < WK; ++t) wn[t] = 32 * t + lane < w.wcap ? __ldg(w.wnode + b * w.wcap + 32 * t + lane) : w.n_nodes;
}

template <int NV, int WK>
__device__ __forceinline__ void issue_warp_nodes(const CatP& c, const double* __restrict__ f, const WarpWinP& w,
                                                 const int (&wn)[WK], int lane, double* nodes, int* wn_s) {
  double2* pr = reinterpret_cast<double2*>(nodes);
  const int wc = w.wcap;
#pragma unroll
  for (int t = 0; t < WK; ++t) {
    const int k = 32 * t + lane;
    if (k < wc) {
      const int node = wn[t];
      wn_s[k] = node;
      if (node < w.n_nodes) {
        const double* xp = c.coords + 4 * (int64_t)node;
        cp_async16(pr + k, xp);
        double* zu = reinterpret_cast<double*>(pr + wc + k);
        cp_async8(zu, xp + 2);
        if constexpr (NV == 6) {
          const double* up = f + 4 * (int64_t)node;
          cp_async8(zu + 1, up);
          double* vw = reinterpret_cast<double*>(pr + 2 * wc + k);
          cp_async8(vw, up + 1);
          cp_async8(vw + 1, up + 2);
        } else {
          cp_async8(zu + 1, f + node);
        }
      }
    }
  }
  cp_async_commit();
}

template <int NN, int NV>
struct WarpSmem {
  static __host__ __device__ size_t node_doubles(int wcap) { return (size_t)NV * wcap; }
  static __host__ __device__ size_t bytes(int wcap) {
    return 2 * node_doubles(wcap) * 8 + (size_t)3 * NN * 32 * 8 + 2 * (size_t)wcap * 4;
  }
};

#ifndef WARP_OCC_K2
#define WARP_OCC_K2 5
#endif
constexpr int kWarpsPerCta = 4;

template <int R, int OP, int WK>
__global__ void __launch_bounds__(kWarpsPerCta * 32, WARP_OCC_K2)
    k_warp(CatP c, WarpWinP w, ab_phys ph, double scale, const double* __restrict__ f, double* __restrict__ out) {
  constexpr int NN = RuleT<R>::NN;
  constexpr int NV = OpT<R, OP>::NV, NC = OpT<R, OP>::NC, STRIDE = OpT<R, OP>::STRIDE;
  using L = WarpSmem<NN, NV>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* mine = smem + (size_t)warp * L::bytes(w.wcap);
  double* nodes0 = reinterpret_cast<double*>(mine);
  double* slots = nodes0 + 2 * L::node_doubles(w.wcap);
  int* wn_s0 = reinterpret_cast<int*>(slots + 3 * NN * 32);
  const int64_t stride = (int64_t)gridDim.x * kWarpsPerCta;
  int64_t b = (int64_t)blockIdx.x * kWarpsPerCta + warp;
  if (b >= w.n_blocks) return;

  LaneRec<NN> rc, rn;
  int wn1[WK], wn2[WK];
  {
    int wn0[WK];
    load_wn<WK>(w, b, lane, wn0);
    issue_warp_nodes<NV, WK>(c, f, w, wn0, lane, nodes0, wn_s0);
  }
  load_rec<NN>(w, b, lane, rc);
  if (b + stride < w.n_blocks) load_wn<WK>(w, b + stride, lane, wn1);

  for (int it = 0; b < w.n_blocks; b += stride, ++it) {
    const int cur = it & 1, nxt = cur ^ 1;
    double* nodes_cur = nodes0 + (size_t)cur * L::node_doubles(w.wcap);
    int* wn_cur = wn_s0 + cur * w.wcap;
    const int64_t b1 = b + stride, b2 = b + 2 * stride;
    if (b1 < w.n_blocks) {
      issue_warp_nodes<NV, WK>(c, f, w, wn1, lane, nodes0 + (size_t)nxt * L::node_doubles(w.wcap),
                               wn_s0 + nxt * w.wcap);
      load_rec<NN>(w, b1, lane, rn);
      if (b2 < w.n_blocks) load_wn<WK>(w, b2, lane, wn2);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    // C: element b*32 + lane from the window -> slots [NC][NN][32]
    const int64_t e = b * 32 + lane;
    if (e < c.n) {
      double x[NN][3], fv[NN][NV == 6 ? 3 : 1];
      const double2* pr = reinterpret_cast<const double2*>(nodes_cur);
      const int wc = w.wcap;
#pragma unroll
      for (int a = 0; a < NN; ++a) {
        const int l = rc.loc[a];
        const double2 xy = pr[l], zf = pr[wc + l];
        x[a][0] = xy.x;
        x[a][1] = xy.y;
        x[a][2] = zf.x;
        fv[a][0] = zf.y;
        if constexpr (NV == 6) {
          const double2 vw = pr[2 * wc + l];
          fv[a][1] = vw.x;
          fv[a][2] = vw.y;
        }
      }
      unwrap<NN>(c, x);
      if constexpr (OP == OP_MOMENTUM) {
        momentum_element<R, NN>(ph, x, fv, [&](int a, const double (&v)[3]) {
#pragma unroll
          for (int k = 0; k < 3; ++k) slots[(k * NN + a) * 32 + lane] = v[k];
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
          for (int k = 0; k < NC; ++k) slots[(k * NN + a) * 32 + lane] = r[a][k];
      }
    } else {
#pragma unroll
      for (int a = 0; a < NN; ++a)
#pragma unroll
        for (int k = 0; k < NC; ++k) slots[(k * NN + a) * 32 + lane] = 0.0;
    }
    __syncwarp();
    // D: segmented sums over the sorted references.  Per-step "add" flags of
    // the shuffle scan depend only on the head bits: computed once.
    const uint32_t h = rc.head;
    const uint32_t nxt_head = __shfl_down_sync(0xffffffffu, h, 1);
    bool fl = h != 0;
    bool add[5];
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const bool up = __shfl_up_sync(0xffffffffu, fl, 1 << s);
      add[s] = lane >= (1 << s) && !fl;
      if (lane >= (1 << s)) fl = fl || up;
    }
    // window index of this lane's first segment: heads before this lane
    int base = __popc(h);
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int up = __shfl_up_sync(0xffffffffu, base, 1 << s);
      if (lane >= (1 << s)) base += up;
    }
    base -= __popc(h);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double sk[NN];
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < NN; ++k) {
        const double v = slots[q * NN * 32 + rc.perm[k]];
        acc = ((h >> k) & 1) ? v : acc + v;
        sk[k] = acc;
      }
      // carry = inclusive segmented sum of the previous lanes' tails
      double cs = acc;
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const double up = __shfl_up_sync(0xffffffffu, cs, 1 << s);
        if (add[s]) cs += up;
      }
      double carry = __shfl_up_sync(0xffffffffu, cs, 1);
      if (lane == 0) carry = 0.0;
      int seg = base - 1;
      bool open = true;  // still inside the segment carried in from the left
#pragma unroll
      for (int k = 0; k < NN; ++k) {
        if ((h >> k) & 1) { open = false; ++seg; }
        const double tot = open ? sk[k] + carry : sk[k];
        const bool end = k < NN - 1 ? ((h >> (k + 1)) & 1) : (lane == 31 || (nxt_head & 1));
        if (end && seg >= 0) {
          const int node = wn_cur[seg];
          if (node < w.n_nodes) red_add(out + (int64_t)node * STRIDE + q, tot);
        }
      }
    }
    __syncwarp();
    rc = rn;
#pragma unroll
    for (int t = 0; t < WK; ++t) wn1[t] = wn2[t];
  }
}

template <int R, int OP, int WK>
static int launch_warp(const CatP& c, const WarpWinP& w, const ab_phys& ph, double scale, const double* f,
                       double* out, cudaStream_t stream) {
  constexpr int NN = RuleT<R>::NN;
  constexpr int NV = OpT<R, OP>::NV;
  const size_t smem = WarpSmem<NN, NV>::bytes(w.wcap) * kWarpsPerCta;
  auto kern = k_warp<R, OP, WK>;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail("warp-window element kernel: shared memory request rejected");
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerCta * 32, smem);
  if (per_sm < 1) return fail("warp-window element kernel does not fit on an SM");
  const int64_t ctas_needed = (w.n_blocks + kWarpsPerCta - 1) / kWarpsPerCta;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > ctas_needed) grid = ctas_needed;
  kern<<<(unsigned)grid, kWarpsPerCta * 32, smem, stream>>>(c, w, ph, scale, f, out);
  return check_launch("k_warp");
}

template <int R, int OP>
static int launch_warp_any(const CatP& c, const WarpWinP& w, const ab_phys& ph, double scale, const double* f,
                           double* out, cudaStream_t stream) {
  switch ((w.wcap + 31) / 32) {
    case 1: return launch_warp<R, OP, 1>(c, w, ph, scale, f, out, stream);
    case 2: return launch_warp<R, OP, 2>(c, w, ph, scale, f, out, stream);
    case 3: return launch_warp<R, OP, 3>(c, w, ph, scale, f, out, stream);
    case 4: return launch_warp<R, OP, 4>(c, w, ph, scale, f, out, stream);
  }
  return fail("warp window wider than 128 nodes");
}
