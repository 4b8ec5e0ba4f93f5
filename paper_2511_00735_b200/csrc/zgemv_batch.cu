// Multi-RHS GEMM for the per-iteration operators (see zgemv_batch.hpp).
//
// Tile: 64 rows x 32 right-hand sides per 256-thread CTA (8 warps as 4 x 2,
// 16 x 16 complex outputs per warp), or 64 x 16 (8 x 1 warps of 8 x 16);
// phases with too few 64-row tiles to fill the SMs (the top levels and the
// coarse matvec: cfg4's coarse matvec ran 88 CTAs) use 32-row tiles on 128
// threads.  K-steps of 16 through a 2-stage cp.async pipeline (3 stages
// measured slower: 15.8 vs 15.5 ms per cfg4 apply; more CTAs per SM win).  The B tile gathers its K rows through the item's index map
// (cp.async with zero-fill for -1 / out-of-range entries), the epilogue
// scatters C rows through theirs.  A complex product is four real DMMAs
// (mma.sync.m8n8k4.f64) on de-interleaved fragments, as in zgemm.cu.
#include "device.cuh"
#include <algorithm>

#include "zgemv_batch.hpp"

namespace hpsb {

namespace {
constexpr int BK = 16;
constexpr int SB = BK + 4;  // complex stride of a B column in smem
template <int BN, int BM>
struct BTile {
  static constexpr int WN = BN / 16, I = BN / 16;       // warp columns; 8-row fragments per warp
  static constexpr int WM = BM / (8 * I);               // warp rows
  static constexpr int THREADS = 32 * WM * WN;          // 256 (BM = 64) or 128 (BM = 32)
  // 64-row tiles: 2 stages (occupancy); 32-row tiles run the phases with few,
  // long tiles (K up to 2816 at one CTA per SM): 4 stages keep more bytes in flight
  static constexpr int STAGES = BM == 32 ? 4 : 2;
  static constexpr int SA = BM + 2;                     // complex stride of an A k-row in smem
  static constexpr int A_STAGE = BK * SA, B_STAGE = BN * SB;
  static constexpr size_t kSmem = sizeof(double2) * STAGES * (A_STAGE + B_STAGE);
};

__device__ __forceinline__ void cpa16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ const double2* bind_ptr(const double2* p, const BBind& b) {
  return !p ? p : p == b.from[0] ? b.to[0] : p == b.from[1] ? b.to[1] : p;
}

// BN = 32 (R > 16): WM x 2 warps of 16 x 16 outputs; BN = 16: WM x 1 warps of 8 x 16.
template <int BN, int BM>
__global__ void __launch_bounds__(BTile<BN, BM>::THREADS) zgemv_batch_kernel(const BDesc* __restrict__ descs,
                                                                              const int* __restrict__ tile_map,
                                                                              int R, BBind bind) {
  using TS = BTile<BN, BM>;
  constexpr int WM = TS::WM, I = TS::I, THREADS = TS::THREADS, SA = TS::SA, STAGES = TS::STAGES;
  constexpr int A_STAGE = TS::A_STAGE, B_STAGE = TS::B_STAGE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As = reinterpret_cast<double2*>(smem_raw);
  double2* Bs = As + STAGES * A_STAGE;
  pdl_trigger();
  const int tile = blockIdx.x;
  BDesc d = descs[tile_map[tile]];
  d.B = bind_ptr(d.B, bind);
  d.C = const_cast<double2*>(bind_ptr(d.C, bind));
  d.Z = bind_ptr(d.Z, bind);
  const int m0 = (tile - d.tile_begin) * BM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int ktiles = d.A ? (d.K + BK - 1) / BK : 0;

  auto load_a = [&](int kt, int st) {
    const int k0 = kt * BK;
    double2* as = As + st * A_STAGE;
#pragma unroll
    for (int r = 0; r < (BM * BK) / THREADS; ++r) {
      const int idx = tid + r * THREADS;
      const int m = idx % BM, k = idx / BM;
      const bool ok = (m0 + m < d.M) && (k0 + k < d.K);
      const double2* src = ok ? d.A + (size_t)(m0 + m) + (size_t)(k0 + k) * d.lda : d.A;
      cpa16(as + k * SA + m, src, ok);
    }
  };
  // B rows are gathered through bidx.  The index of a stage is loaded one
  // k-step ahead (rows_of) and kept in registers: loaded inside load_b, every
  // k-step stalled on an L2 round trip before its copies could be issued
  // (2 us per step at one CTA per SM: cfg4's coarse matvec ran at 0.7 TB/s).
  constexpr int NB = (BN * BK) / THREADS;
  auto rows_of = [&](int kt, int (&rows)[NB]) {
    const int k0 = kt * BK;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      const int k = (tid + r * THREADS) % BK;
      rows[r] = k0 + k < d.K ? (d.bidx ? __ldg(d.bidx + k0 + k) : k0 + k) : -1;
    }
  };
  auto load_b = [&](int st, const int (&rows)[NB]) {
    double2* bs = Bs + st * B_STAGE;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      const int idx = tid + r * THREADS;
      const int k = idx % BK, n = idx / BK;
      const bool ok = n < R && rows[r] >= 0;
      const double2* src = ok ? d.B + (size_t)rows[r] + (size_t)n * d.ldb : d.B;
      cpa16(bs + n * SB + k, src, ok);
    }
  };

  double cr[I][2][2], ci[I][2][2];
#pragma unroll
  for (int i = 0; i < I; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

  // operators are static: their first stages are issued before the PDL wait
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s)
    if (s < ktiles) load_a(s, s);
  int brow[NB];
  pdl_wait();
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) {
      rows_of(s, brow);
      load_b(s, brow);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  if (STAGES - 1 < ktiles) rows_of(STAGES - 1, brow);
  const int arow = wm * (8 * I) + (lane >> 2), kq = lane & 3;
  const int bcol = wn * 16 + (lane >> 2);
  for (int kt = 0; kt < ktiles; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 2));
    __syncthreads();
    if (kt + STAGES - 1 < ktiles) {
      load_a(kt + STAGES - 1, (kt + STAGES - 1) % STAGES);
      load_b((kt + STAGES - 1) % STAGES, brow);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    if (kt + STAGES < ktiles) rows_of(kt + STAGES, brow);  // next step's rows: the load overlaps the DMMAs below
    const double2* as = As + (kt % STAGES) * A_STAGE;
    const double2* bs = Bs + (kt % STAGES) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double2 a[I], b[2];
#pragma unroll
      for (int i = 0; i < I; ++i) a[i] = as[(kk + kq) * SA + arow + i * 8];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = bs[(bcol + j * 8) * SB + kk + kq];
      // four passes over the I x 2 fragment grid: the two DMMAs into the
      // same accumulator are 2 I issues apart instead of back to back (the
      // asm statements are volatile, so the compiler keeps this order)
#pragma unroll
      for (int i = 0; i < I; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
#pragma unroll
      for (int i = 0; i < I; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(ci[i][j][0], ci[i][j][1], a[i].x, b[j].y);
#pragma unroll
      for (int i = 0; i < I; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(cr[i][j][0], cr[i][j][1], -a[i].y, b[j].y);
#pragma unroll
      for (int i = 0; i < I; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(ci[i][j][0], ci[i][j][1], a[i].y, b[j].x);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  // epilogue: C[cidx[m], n] = alpha acc + gamma Z[zidx[m], n] + beta C[cidx[m], n]
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const int row = m0 + wm * (8 * I) + i * 8 + (lane >> 2);
    if (row >= d.M) continue;
    const int crow = d.cidx ? __ldg(d.cidx + row) : row;
    if (crow < 0) continue;
    const int zrow = d.gamma != 0.0 ? (d.zidx ? __ldg(d.zidx + row) : row) : -1;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = wn * 16 + j * 8 + 2 * (lane & 3) + h;
        if (col >= R) continue;
        double2* c = d.C + (size_t)crow + (size_t)col * d.ldc;
        double2 v = cscale(make_double2(cr[i][j][h], ci[i][j][h]), d.alpha);
        if (zrow >= 0) v = cadd(v, cscale(__ldcg(d.Z + (size_t)zrow + (size_t)col * d.ldz), d.gamma));
        if (d.beta != 0.0) v = cadd(v, cscale(__ldcg(c), d.beta));
        __stcg(c, v);
      }
  }
}
}  // namespace

void BPhase::add(const BDesc& x0) {
  if (x0.M <= 0) return;
  if (x0.A) {
    flops += 8.0 * x0.M * x0.K;  // per right-hand side
    bytes += 16.0 * x0.M * x0.K;
  }
  descs.push_back(x0);
}

void BPhase::finalize(cudaStream_t s) {
  // 32-row tiles when 64-row tiles would leave SMs without a CTA
  int tiles64 = 0;
  for (const BDesc& x : descs) tiles64 += (x.M + 63) / 64;
  bm = tiles64 < 2 * 148 ? 32 : 64;
  total_tiles = 0;
  for (BDesc& x : descs) {
    x.tiles_m = (x.M + bm - 1) / bm;
    x.tile_begin = total_tiles;
    total_tiles += x.tiles_m;
  }
  d.upload(descs, s);
  std::vector<int> map(total_tiles);
  for (size_t i = 0; i < descs.size(); ++i) {
    const int end = i + 1 < descs.size() ? descs[i + 1].tile_begin : total_tiles;
    std::fill(map.begin() + descs[i].tile_begin, map.begin() + end, static_cast<int>(i));
  }
  d_map.upload(map, s);
}

namespace {
template <int BN, int BM>
void launch_batch(Context* ctx, int tiles, const BDesc* descs, const int* map, int R, const BBind& bind) {
  using TS = BTile<BN, BM>;
  allow_smem<zgemv_batch_kernel<BN, BM>>(TS::kSmem);
  launch_k(ctx, zgemv_batch_kernel<BN, BM>, dim3(tiles), dim3(TS::THREADS), TS::kSmem, 1, descs, map, R, bind);
}
}  // namespace

void BPhase::run(Context* ctx, int R, const char* label, BBind bind) const {
  if (descs.empty()) return;
  if (R < 1 || R > kBatchMaxRhs) throw InvalidArgument("batch: 1 <= nrhs <= 32");
  KernelScope ks(ctx, this->label.empty() ? label : this->label.c_str(), bytes, flops * R);
  const BDesc* dp = d.p;
  const int* mp = d_map.p;
  if (R <= 16) {
    if (bm == 32) launch_batch<16, 32>(ctx, total_tiles, dp, mp, R, bind);
    else launch_batch<16, 64>(ctx, total_tiles, dp, mp, R, bind);
  } else {
    if (bm == 32) launch_batch<32, 32>(ctx, total_tiles, dp, mp, R, bind);
    else launch_batch<32, 64>(ctx, total_tiles, dp, mp, R, bind);
  }
}

}  // namespace hpsb
