// Microbenchmark: streaming k basis vectors of n doubles, separate (strided)
// vs chunk-blocked layouts, plain loads vs TMA bulk copies.  Informs the
// Krylov basis layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_1906_04051_b200/csrc/tma.cuh"

using namespace pgm;

constexpr int CHR = 256;

// out[row] = sum_l V_l[row]; separate layout, plain loads
__global__ void k_plain_sep(const double* __restrict__ V, size_t ld, int k, int n, double* out) {
  for (size_t row = blockIdx.x * (size_t)blockDim.x + threadIdx.x; row < (size_t)n;
       row += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int l = 0; l < k; ++l) s += V[l * ld + row];
    out[row] = s;
  }
}

// blocked layout: V[c][l][i], chunk stride k*CHR
__global__ void k_plain_blk(const double* __restrict__ V, int k, int n, double* out) {
  const int nch = (n + CHR - 1) / CHR;
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const double* base = V + (size_t)c * k * CHR;
    const int i = threadIdx.x;
    double s = 0.0;
#pragma unroll 8
    for (int l = 0; l < k; ++l) s += base[l * CHR + i];
    if (c * CHR + i < n) out[c * CHR + i] = s;
  }
}

// TMA pipeline, separate (k copies per chunk) or blocked (1 copy per chunk)
template <bool BLOCKED>
__global__ void k_tma(const double* __restrict__ V, size_t ld, int k, int n, double* out,
                      int nstages) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  double* st = sm + 16;
  const size_t ssz = (size_t)k * CHR;
  const int nch = (n + CHR - 1) / CHR;
  const int my = (int)blockIdx.x < nch ? (nch - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int s = i % nstages;
    const size_t c = blockIdx.x + (size_t)i * gridDim.x;
    if (lane == 0) mbar_arrive_expect_tx(&bars[s], (uint32_t)(k * CHR * 8));
    __syncwarp();
    if (BLOCKED) {
      if (lane == 0) tma_load_1d(st + s * ssz, V + c * k * CHR, k * CHR * 8, &bars[s]);
    } else {
      for (int l = lane; l < k; l += 32)
        tma_load_1d(st + s * ssz + (size_t)l * CHR, V + l * ld + c * CHR, CHR * 8, &bars[s]);
    }
  };
  if (warp == 0)
    for (int i = 0; i < min(nstages, my); ++i) issue(i);
  for (int i = 0; i < my; ++i) {
    const int s = i % nstages;
    mbar_wait(&bars[s], (i / nstages) & 1);
    const double* b = st + s * ssz;
    double acc = 0.0;
    for (int l = 0; l < k; ++l) acc += b[l * CHR + tid];
    const size_t c = blockIdx.x + (size_t)i * gridDim.x;
    if (c * CHR + tid < (size_t)n) out[c * CHR + tid] = acc;
    __syncthreads();
    if (warp == 0 && i + nstages < my) issue(i + nstages);
  }
}

int main() {
  const int n = 1030301, kmax = 51;
  const size_t ld = ((n + 256 + 127) / 128) * 128;
  double *V, *out;
  cudaMalloc(&V, sizeof(double) * ld * kmax);
  cudaMalloc(&out, sizeof(double) * ld);
  cudaMemset(V, 0, sizeof(double) * ld * kmax);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    const int R = 20;
    for (int r = 0; r < R; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / R;
  };
  for (int k : {4, 13, 26, 51}) {
    const double bytes = 8.0 * n * (k + 1);
    float t1 = timeit([&] { k_plain_sep<<<nsm * 8, 256>>>(V, ld, k, n, out); });
    float t2 = timeit([&] { k_plain_blk<<<nsm * 8, CHR>>>(V, k, n, out); });
    const size_t stage = (size_t)k * CHR * 8;
    int S = (int)std::min<size_t>(8, (200 * 1024) / stage);
    if (S < 2) S = 2;
    const size_t smem = 128 + S * stage;
    cudaFuncSetAttribute(k_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float t3 = timeit([&] { k_tma<false><<<nsm, CHR, smem>>>(V, ld, k, n, out, S); });
    float t4 = timeit([&] { k_tma<true><<<nsm, CHR, smem>>>(V, ld, k, n, out, S); });
    // 2 blocks / SM variant with half the stages
    int S2 = std::max(2, S / 2);
    const size_t smem2 = 128 + S2 * stage;
    float t5 = timeit([&] { k_tma<true><<<nsm * 2, CHR, smem2>>>(V, ld, k, n, out, S2); });
    printf("k=%2d  plain_sep %7.1f  plain_blk %7.1f  tma_sep %7.1f  tma_blk %7.1f  tma_blk_2x %7.1f GB/s (S=%d)\n",
           k, bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t3 / 1e6, bytes / t4 / 1e6,
           bytes / t5 / 1e6, S);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
