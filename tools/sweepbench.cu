// Microbenchmark of the CGS2 sweep kernel designs.
//   pass B: w1 = w + sum_l a_l V_l ; h_l = V_l . w1   (l < NP)
//   pass C: w2 = w1 + sum_l b_l V_l ; ||w2||^2, U_j . w2 (j < r)
// Variants differ in how the per-row products are reduced:
//   B0/C0: per-chunk warp transpose through smem (the library's first design)
//   B1   : lane-private register accumulators across chunks, one reduction at the end
//   B2   : lane-private accumulators in smem (LDS/DFMA/STS per value)
//   C1   : U loads issued with the V loads, lane-private register accumulators
//   S    : plain streaming upper bound (same loads, out = sum)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sweepbench tools/sweepbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1906_04051_b200/csrc/tma.cuh"

using namespace pgm;

constexpr int BLK = 128;
constexpr int WPB = BLK / 32;
constexpr int TPS = 33;

struct Args {
  const double* V;
  double* w;
  const double* U;
  const double* a;
  int r;
  int n;
  size_t ld;
  double* part;  // [grid][64]
};

__device__ __forceinline__ void prefetch_chunk(const Args& A, int np, int nu, int c, int lane) {
  const size_t off = (size_t)c * 32;
  for (int q = lane; q < np + 1 + nu; q += 32) {
    const double* src = q < np ? A.V + (size_t)q * A.ld : (q == np ? A.w : A.U + (size_t)(q - np - 1) * A.ld);
    tma_prefetch_l2(src + off, 256);
  }
}

// block-level final reduction of per-lane values vals[NV] -> part[blockIdx][NV]
template <int NV>
__device__ __forceinline__ void block_out(const Args& A, const double (&vals)[NV], double* sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warp sums via shuffles (end-of-kernel only)
  for (int v = 0; v < NV; ++v) {
    double s = vals[v];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sm[warp * 64 + v] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < WPB; ++w) s += sm[w * 64 + threadIdx.x];
    A.part[blockIdx.x * 64 + threadIdx.x] = s;
  }
}

// ---- S: streaming upper bound
template <int NP>
__global__ void __launch_bounds__(BLK) k_S(Args A) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (A.n + 31) >> 5, W = gridDim.x * WPB;
  for (int c = blockIdx.x * WPB + warp; c < nch; c += W) {
    const int row = c * 32 + lane;
    double v[NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) v[l] = __ldg(A.V + (size_t)l * A.ld + row);
    double o = A.w[row];
    __syncwarp();
#pragma unroll
    for (int l = 0; l < NP; ++l) o += v[l];
    A.w[row] = o;
  }
}

// ---- B0: per-chunk transpose (library design)
template <int NP>
__global__ void __launch_bounds__(BLK) k_B0(Args A) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tp = sm + warp * 16 * TPS;
  const int nch = (A.n + 31) >> 5, W = gridDim.x * WPB;
  constexpr int NS = (NP + 15) / 16;
  double acc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) acc[s] = 0.0;
  prefetch_chunk(A, NP, 0, blockIdx.x * WPB + warp, lane);
  for (int c = blockIdx.x * WPB + warp; c < nch; c += W) {
    if (c + W < nch) prefetch_chunk(A, NP, 0, c + W, lane);
    const int row = c * 32 + lane;
    double v[NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) v[l] = __ldg(A.V + (size_t)l * A.ld + row);
    const double win = A.w[row];
    __syncwarp();
    double o4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int l = 0; l < NP; ++l) o4[l & 3] += A.a[l] * v[l];
    const double o = win + ((o4[0] + o4[1]) + (o4[2] + o4[3]));
    A.w[row] = o;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int cnt = (NP - s * 16) < 16 ? (NP - s * 16) : 16;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < cnt) tp[j * TPS + lane] = v[s * 16 + j < NP ? s * 16 + j : 0] * o;
      __syncwarp();
      const double* p = tp + (lane & 15) * TPS + (lane >> 4) * 16;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
      for (int q = 0; q < 16; q += 4) {
        a0 += p[q];
        a1 += p[q + 1];
        a2 += p[q + 2];
        a3 += p[q + 3];
      }
      double t = (a0 + a1) + (a2 + a3);
      t += __shfl_xor_sync(0xffffffffu, t, 16);
      if (lane < cnt) acc[s] += t;
      __syncwarp();
    }
  }
  __syncthreads();
  // lane l of slot s holds value s*16+l: spread to a per-lane array
  double vals[NP];
#pragma unroll
  for (int l = 0; l < NP; ++l) vals[l] = 0.0;
  (void)vals;
  if (lane < 16)
    for (int s = 0; s < NS; ++s)
      if (s * 16 + lane < NP) sm[(WPB * 16 * TPS) + warp * 64 + s * 16 + lane] = acc[s];
  __syncthreads();
  if (threadIdx.x < NP) {
    double s = 0.0;
    for (int w = 0; w < WPB; ++w) s += sm[(WPB * 16 * TPS) + w * 64 + threadIdx.x];
    A.part[blockIdx.x * 64 + threadIdx.x] = s;
  }
}

// ---- B1: lane-private register accumulators
template <int NP>
__global__ void __launch_bounds__(BLK) k_B1(Args A) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (A.n + 31) >> 5, W = gridDim.x * WPB;
  double acc[NP];
#pragma unroll
  for (int l = 0; l < NP; ++l) acc[l] = 0.0;
  prefetch_chunk(A, NP, 0, blockIdx.x * WPB + warp, lane);
  for (int c = blockIdx.x * WPB + warp; c < nch; c += W) {
    if (c + W < nch) prefetch_chunk(A, NP, 0, c + W, lane);
    const int row = c * 32 + lane;
    double v[NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) v[l] = __ldg(A.V + (size_t)l * A.ld + row);
    const double win = A.w[row];
    __syncwarp();
    double o4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int l = 0; l < NP; ++l) o4[l & 3] += A.a[l] * v[l];
    const double o = win + ((o4[0] + o4[1]) + (o4[2] + o4[3]));
    A.w[row] = o;
#pragma unroll
    for (int l = 0; l < NP; ++l) acc[l] += v[l] * o;
  }
  block_out<NP>(A, acc, sm);
}

// ---- B2: lane-private accumulators in smem
template <int NP>
__global__ void __launch_bounds__(BLK) k_B2(Args A) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* acc = sm + 64 * WPB + warp * NP * 32 + lane;
  const int nch = (A.n + 31) >> 5, W = gridDim.x * WPB;
#pragma unroll
  for (int l = 0; l < NP; ++l) acc[l * 32] = 0.0;
  prefetch_chunk(A, NP, 0, blockIdx.x * WPB + warp, lane);
  for (int c = blockIdx.x * WPB + warp; c < nch; c += W) {
    if (c + W < nch) prefetch_chunk(A, NP, 0, c + W, lane);
    const int row = c * 32 + lane;
    double v[NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) v[l] = __ldg(A.V + (size_t)l * A.ld + row);
    const double win = A.w[row];
    __syncwarp();
    double o4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int l = 0; l < NP; ++l) o4[l & 3] += A.a[l] * v[l];
    const double o = win + ((o4[0] + o4[1]) + (o4[2] + o4[3]));
    A.w[row] = o;
#pragma unroll
    for (int l = 0; l < NP; ++l) acc[l * 32] += v[l] * o;
  }
  double vals[1];
  (void)vals;
  __syncthreads();
  if (threadIdx.x < NP) {
    double s = 0.0;
    for (int w = 0; w < WPB; ++w)
      for (int ln = 0; ln < 32; ++ln) s += sm[64 * WPB + w * NP * 32 + threadIdx.x * 32 + ln];
    A.part[blockIdx.x * 64 + threadIdx.x] = s;
  }
}

// ---- C0: library design (dots with U read after o)
template <int NP>
__global__ void __launch_bounds__(BLK) k_C0(Args A) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tp = sm + warp * 16 * TPS;
  const int nch = (A.n + 31) >> 5, W = gridDim.x * WPB;
  const int nv = 1 + A.r;
  double acc[2] = {0, 0};
  prefetch_chunk(A, NP, A.r, blockIdx.x * WPB + warp, lane);
  for (int c = blockIdx.x * WPB + warp; c < nch; c += W) {
    if (c + W < nch) prefetch_chunk(A, NP, A.r, c + W, lane);
    const int row = c * 32 + lane;
    double v[NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) v[l] = __ldg(A.V + (size_t)l * A.ld + row);
    const double win = A.w[row];
    __syncwarp();
    double o4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int l = 0; l < NP; ++l) o4[l & 3] += A.a[l] * v[l];
    const double o = win + ((o4[0] + o4[1]) + (o4[2] + o4[3]));
    A.w[row] = o;
    for (int s = 0; s < 2; ++s) {
      if (s * 16 >= nv) break;
      const int cnt = min(16, nv - s * 16);
      double p[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int vv = s * 16 + j;
        p[j] = j < cnt ? (vv == 0 ? o * o : __ldg(A.U + (size_t)(vv - 1) * A.ld + row) * o) : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < cnt) tp[j * TPS + lane] = p[j];
      __syncwarp();
      const double* q = tp + (lane & 15) * TPS + (lane >> 4) * 16;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
      for (int t = 0; t < 16; t += 4) {
        a0 += q[t];
        a1 += q[t + 1];
        a2 += q[t + 2];
        a3 += q[t + 3];
      }
      double t = (a0 + a1) + (a2 + a3);
      t += __shfl_xor_sync(0xffffffffu, t, 16);
      if (lane < cnt) acc[s] += t;
      __syncwarp();
    }
  }
  __syncthreads();
  if (lane < 16)
    for (int s = 0; s < 2; ++s)
      if (s * 16 + lane < nv) sm[(WPB * 16 * TPS) + warp * 64 + s * 16 + lane] = acc[s];
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int w = 0; w < WPB; ++w) s += sm[(WPB * 16 * TPS) + w * 64 + threadIdx.x];
    A.part[blockIdx.x * 64 + threadIdx.x] = s;
  }
}

// ---- C1: U loads issued with the V loads; lane-private register accumulators
template <int NP, int RMAX>
__global__ void __launch_bounds__(BLK) k_C1(Args A) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (A.n + 31) >> 5, W = gridDim.x * WPB;
  const int r = A.r;
  double acc[1 + RMAX];
#pragma unroll
  for (int l = 0; l <= RMAX; ++l) acc[l] = 0.0;
  prefetch_chunk(A, NP, r, blockIdx.x * WPB + warp, lane);
  for (int c = blockIdx.x * WPB + warp; c < nch; c += W) {
    if (c + W < nch) prefetch_chunk(A, NP, r, c + W, lane);
    const int row = c * 32 + lane;
    double v[NP], u[RMAX];
#pragma unroll
    for (int l = 0; l < NP; ++l) v[l] = __ldg(A.V + (size_t)l * A.ld + row);
#pragma unroll
    for (int l = 0; l < RMAX; ++l) u[l] = l < r ? __ldg(A.U + (size_t)l * A.ld + row) : 0.0;
    const double win = A.w[row];
    __syncwarp();
    double o4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int l = 0; l < NP; ++l) o4[l & 3] += A.a[l] * v[l];
    const double o = win + ((o4[0] + o4[1]) + (o4[2] + o4[3]));
    A.w[row] = o;
    acc[0] += o * o;
#pragma unroll
    for (int l = 0; l < RMAX; ++l) acc[1 + l] += u[l] * o;
  }
  block_out<1 + RMAX>(A, acc, sm);
}

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

template <class K>
float timeit(K kern, const Args& A, size_t smem, int reps) {
  int occ = 0;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BLK, smem));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int nch = (A.n + 31) / 32;
  const int G = std::min((nch + WPB - 1) / WPB, occ * nsm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) kern<<<G, BLK, smem>>>(A);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) kern<<<G, BLK, smem>>>(A);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  printf("  [occ %d regs %d] ", occ, fa.numRegs);
  return ms / reps;
}


// ---- B3/C3: vector set split across the NW warps of a block; all warps work
// on the same 32-row chunk, partial row sums combined through smem (one
// barrier per chunk, double-buffered); lane-private register accumulators.
template <int NP, int NW, bool DB, bool MODEC, int RMAX>
__global__ void __launch_bounds__(NW * 32) k_split(Args A) {
  __shared__ double red[2][NW][32];
  __shared__ double fin[NW][RMAX + NP / NW + 2];
  constexpr int NPW = (NP + NW - 1) / NW;
  constexpr int NUW = MODEC ? (RMAX + NW - 1) / NW : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (A.n + 31) >> 5;
  const int r = A.r;
  double acc[MODEC ? NUW + 1 : NPW];
#pragma unroll
  for (int j = 0; j < (MODEC ? NUW + 1 : NPW); ++j) acc[j] = 0.0;
  double aw[NPW];
#pragma unroll
  for (int j = 0; j < NPW; ++j) aw[j] = (warp + NW * j < NP) ? A.a[warp + NW * j] : 0.0;
  double v[NPW], u[NUW > 0 ? NUW : 1], win = 0.0;
  auto load = [&](int c, double (&vv)[NPW], double (&uu)[NUW > 0 ? NUW : 1], double& ww) {
    const int row = c * 32 + lane;
#pragma unroll
    for (int j = 0; j < NPW; ++j)
      vv[j] = (warp + NW * j < NP) ? __ldg(A.V + (size_t)(warp + NW * j) * A.ld + row) : 0.0;
    if (MODEC) {
#pragma unroll
      for (int j = 0; j < NUW; ++j)
        uu[j] = (warp + NW * j < r) ? __ldg(A.U + (size_t)(warp + NW * j) * A.ld + row) : 0.0;
    }
    ww = warp == 0 ? A.w[row] : 0.0;
  };
  int c = blockIdx.x;
  if (c < nch) load(c, v, u, win);
  int buf = 0;
  for (; c < nch; c += gridDim.x) {
    // prefetch the chunk after next into L2 (one 256 B segment per lane)
    {
      const int cp = c + 2 * gridDim.x;
      if (cp < nch) {
        const size_t off = (size_t)cp * 32;
        for (int q = lane; q < NPW + NUW + 1; q += 32) {
          const int l = warp + NW * q;
          if (q < NPW) { if (l < NP) tma_prefetch_l2(A.V + (size_t)l * A.ld + off, 256); }
          else if (q < NPW + NUW) { const int lu = warp + NW * (q - NPW); if (lu < r) tma_prefetch_l2(A.U + (size_t)lu * A.ld + off, 256); }
          else if (warp == 0) tma_prefetch_l2(A.w + off, 256);
        }
      }
    }
    double p4[2] = {win, 0.0};
#pragma unroll
    for (int j = 0; j < NPW; ++j) p4[j & 1] += aw[j] * v[j];
    red[buf][warp][lane] = p4[0] + p4[1];
    double vn[NPW], un[NUW > 0 ? NUW : 1], wn = 0.0;
    if (DB && c + (int)gridDim.x < nch) load(c + gridDim.x, vn, un, wn);
    __syncthreads();
    double o = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) o += red[buf][w][lane];
    const int row = c * 32 + lane;
    if (warp == 0) A.w[row] = o;
    if (!MODEC) {
#pragma unroll
      for (int j = 0; j < NPW; ++j) acc[j] += v[j] * o;
    } else {
      if (warp == 0) acc[NUW] += o * o;
#pragma unroll
      for (int j = 0; j < NUW; ++j) acc[j] += u[j] * o;
    }
    if (DB) {
#pragma unroll
      for (int j = 0; j < NPW; ++j) v[j] = vn[j];
#pragma unroll
      for (int j = 0; j < NUW; ++j) u[j] = un[j];
      win = wn;
    } else if (c + (int)gridDim.x < nch) {
      load(c + gridDim.x, v, u, win);
    }
    buf ^= 1;
  }
  // end: warp sums of the lane-private accumulators
  constexpr int NA = MODEC ? NUW + 1 : NPW;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    double s = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) fin[warp][j] = s;
  }
  __syncthreads();
  if (threadIdx.x < NW * NA) {
    const int w = threadIdx.x % NW, j = threadIdx.x / NW;
    A.part[blockIdx.x * 64 + (w + NW * j) % 64] = fin[w][j];
  }
}

template <class K>
float timeit_grid(K kern, const Args& A, int threads, int reps) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int nch = (A.n + 31) / 32;
  const int G = std::min(nch, occ * nsm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) kern<<<G, threads>>>(A);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) kern<<<G, threads>>>(A);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  printf("  [occ %d regs %d] ", occ, fa.numRegs);
  return ms / reps;
}

// B4/C4: as k_split but every lane owns 2 consecutive rows (double2 loads, 64-row chunks)
template <int NP, int NW, bool MODEC, int RMAX>
__global__ void __launch_bounds__(NW * 32) k_split2(Args A) {
  __shared__ double2 red[2][NW][32];
  __shared__ double fin[NW][RMAX + NP / NW + 2];
  constexpr int NPW = (NP + NW - 1) / NW;
  constexpr int NUW = MODEC ? (RMAX + NW - 1) / NW : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (A.n + 63) >> 6;
  const int r = A.r;
  double acc[MODEC ? NUW + 1 : NPW];
#pragma unroll
  for (int j = 0; j < (MODEC ? NUW + 1 : NPW); ++j) acc[j] = 0.0;
  double aw[NPW];
#pragma unroll
  for (int j = 0; j < NPW; ++j) aw[j] = (warp + NW * j < NP) ? A.a[warp + NW * j] : 0.0;
  int buf = 0;
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const int cp = c + gridDim.x;
    if (cp < nch) {
      const size_t off = (size_t)cp * 64;
      for (int q = lane; q < NPW + NUW + 1; q += 32) {
        const int l = warp + NW * q;
        if (q < NPW) { if (l < NP) tma_prefetch_l2(A.V + (size_t)l * A.ld + off, 512); }
        else if (q < NPW + NUW) { const int lu = warp + NW * (q - NPW); if (lu < r) tma_prefetch_l2(A.U + (size_t)lu * A.ld + off, 512); }
        else if (warp == 0) tma_prefetch_l2(A.w + off, 512);
      }
    }
    const size_t row = (size_t)c * 64 + 2 * lane;
    double2 v[NPW], u[NUW > 0 ? NUW : 1];
#pragma unroll
    for (int j = 0; j < NPW; ++j)
      v[j] = (warp + NW * j < NP) ? __ldg(reinterpret_cast<const double2*>(A.V + (size_t)(warp + NW * j) * A.ld + row)) : make_double2(0, 0);
    if (MODEC) {
#pragma unroll
      for (int j = 0; j < NUW; ++j)
        u[j] = (warp + NW * j < r) ? __ldg(reinterpret_cast<const double2*>(A.U + (size_t)(warp + NW * j) * A.ld + row)) : make_double2(0, 0);
    }
    double2 win = warp == 0 ? *reinterpret_cast<const double2*>(A.w + row) : make_double2(0, 0);
    __syncwarp();
    double2 p = win;
#pragma unroll
    for (int j = 0; j < NPW; ++j) { p.x += aw[j] * v[j].x; p.y += aw[j] * v[j].y; }
    red[buf][warp][lane] = p;
    __syncthreads();
    double2 o = make_double2(0, 0);
#pragma unroll
    for (int w = 0; w < NW; ++w) { const double2 t = red[buf][w][lane]; o.x += t.x; o.y += t.y; }
    if (warp == 0) *reinterpret_cast<double2*>(A.w + row) = o;
    if (!MODEC) {
#pragma unroll
      for (int j = 0; j < NPW; ++j) acc[j] += v[j].x * o.x + v[j].y * o.y;
    } else {
      if (warp == 0) acc[NUW] += o.x * o.x + o.y * o.y;
#pragma unroll
      for (int j = 0; j < NUW; ++j) acc[j] += u[j].x * o.x + u[j].y * o.y;
    }
    buf ^= 1;
  }
  constexpr int NA = MODEC ? NUW + 1 : NPW;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    double s = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) fin[warp][j] = s;
  }
  __syncthreads();
  if (threadIdx.x < NW * NA) {
    const int w = threadIdx.x % NW, j = threadIdx.x / NW;
    A.part[blockIdx.x * 64 + (w + NW * j) % 64] = fin[w][j];
  }
}

template <int NP>
void run(const Args& A0, int r) {
  Args A = A0;
  A.r = r;
  const double n = A.n;
  const double bytesB = 8.0 * n * (NP + 2);
  const double bytesC = 8.0 * n * (NP + 2 + r);
  const int reps = 20;
  float t;
  printf("NP=%d r=%d\n", NP, r);
  t = timeit(k_S<NP>, A, 0, reps);
  printf("S   %8.1f us %7.0f GB/s\n", t * 1e3, bytesB / (t * 1e-3) / 1e9);
  t = timeit(k_B0<NP>, A, 8 * (WPB * 16 * TPS + WPB * 64), reps);
  printf("B0  %8.1f us %7.0f GB/s\n", t * 1e3, bytesB / (t * 1e-3) / 1e9);
  t = timeit(k_B1<NP>, A, 8 * (WPB * 64), reps);
  printf("B1  %8.1f us %7.0f GB/s\n", t * 1e3, bytesB / (t * 1e-3) / 1e9);
  t = timeit(k_B2<NP>, A, 8 * (WPB * 64 + WPB * NP * 32), reps);
  printf("B2  %8.1f us %7.0f GB/s\n", t * 1e3, bytesB / (t * 1e-3) / 1e9);
  t = timeit(k_C0<NP>, A, 8 * (WPB * 16 * TPS + WPB * 64), reps);
  printf("C0  %8.1f us %7.0f GB/s\n", t * 1e3, bytesC / (t * 1e-3) / 1e9);
  t = timeit(k_C1<NP, 8>, A, 8 * (WPB * 64), reps);
  printf("C1/8  %8.1f us %7.0f GB/s\n", t * 1e3, bytesC / (t * 1e-3) / 1e9);
  t = timeit(k_C1<NP, 20>, A, 8 * (WPB * 64), reps);
  printf("C1/20 %8.1f us %7.0f GB/s\n", t * 1e3, bytesC / (t * 1e-3) / 1e9);

#define SPL(NW, DB) \
  t = timeit_grid(k_split<NP, NW, DB, false, 20>, A, NW * 32, reps); \
  printf("B3/%d%s %8.1f us %7.0f GB/s\n", NW, DB ? "db" : "", t * 1e3, bytesB / (t * 1e-3) / 1e9); \
  t = timeit_grid(k_split<NP, NW, DB, true, 20>, A, NW * 32, reps); \
  printf("C3/%d%s %8.1f us %7.0f GB/s\n", NW, DB ? "db" : "", t * 1e3, bytesC / (t * 1e-3) / 1e9);
  SPL(2, false) SPL(4, false) SPL(4, true) SPL(8, false)
#define SPL2(NW) \
  t = timeit_grid(k_split2<NP, NW, false, 20>, A, NW * 32, reps); \
  printf("B4/%d %8.1f us %7.0f GB/s\n", NW, t * 1e3, bytesB / (t * 1e-3) / 1e9); \
  t = timeit_grid(k_split2<NP, NW, true, 20>, A, NW * 32, reps); \
  printf("C4/%d %8.1f us %7.0f GB/s\n", NW, t * 1e3, bytesC / (t * 1e-3) / 1e9);
  SPL2(2) SPL2(4) SPL2(8)
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1030301;
  const size_t ld = ((size_t)n + 256 + 127) / 128 * 128;
  Args A{};
  double *V, *w, *U, *a, *part;
  CK(cudaMalloc(&V, 52 * ld * 8));
  CK(cudaMalloc(&w, ld * 8));
  CK(cudaMalloc(&U, 21 * ld * 8));
  CK(cudaMalloc(&a, 64 * 8));
  CK(cudaMalloc(&part, 64 * 8 * 148 * 64));
  CK(cudaMemset(V, 0, 52 * ld * 8));
  CK(cudaMemset(w, 0, ld * 8));
  CK(cudaMemset(U, 0, 21 * ld * 8));
  CK(cudaMemset(a, 0, 64 * 8));
  A.V = V;
  A.w = w;
  A.U = U;
  A.a = a;
  A.n = n;
  A.ld = ld;
  A.part = part;
  run<1>(A, 5);
  run<4>(A, 5);
  run<8>(A, 5);
  run<16>(A, 5);
  run<26>(A, 5);
  run<26>(A, 20);
  run<40>(A, 5);
  run<51>(A, 5);
  return 0;
}
