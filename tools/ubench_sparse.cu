// ubench_sparse.cu -- microbenchmarks that size the sparse-term (a4) inner loop
// on sm_100a: FMA-pipe variants and the smem-gather + FMA loop shapes.
// Reports MAC per clock per SM from in-kernel clock64 (clock-independent).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_sparse.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__device__ unsigned long long g_cycles[4096];

// ---- pure pipe throughput: 16 independent chains per thread
__global__ void k_ffma(float* out, float a, int iters) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float b = a * 0.5f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float* out, float a, int iters) {
  unsigned long long acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 f = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    acc[i] = *reinterpret_cast<unsigned long long*>(&f);
  }
  float2 af = make_float2(a, a), bf = make_float2(a * 0.5f, a * 0.25f);
  unsigned long long av = *reinterpret_cast<unsigned long long*>(&af);
  unsigned long long bv = *reinterpret_cast<unsigned long long*>(&bf);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(av), "l"(bv));
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 f = *reinterpret_cast<float2*>(&acc[i]);
    s += f.x + f.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// mixed precision fma: f32 += bf16 * bf16 (FHFMA.BF16 with H0/H1 selectors)
__global__ void k_fhfma(float* out, float a, int iters) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  __nv_bfloat162 xv = __floats2bfloat162_rn(a, a * 0.5f);
  uint32_t x = *reinterpret_cast<uint32_t*>(&xv);
  uint32_t w = x ^ 0x00010001u;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile(
          "{\n\t.reg .b16 l, h, wl, wh;\n\tmov.b32 {l,h}, %2;\n\tmov.b32 {wl,wh}, %3;\n\t"
          "fma.rn.f32.bf16 %0, l, wl, %0;\n\t"
          "fma.rn.f32.bf16 %1, h, wl, %1;\n\t}"
          : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1])
          : "r"(x), "r"(w));
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// ---- the sparse-term inner loop shapes.  smem: a "window" of 16-byte vectors
// (8 bf16 images or 4 fp32 images) + a metadata list of packed nonzeros.
// Each thread owns a base vector slot; each nonzero = (bf16 value | u16 byte offset << 16).
constexpr int kWinBytes = 96 * 1024;
constexpr int kMeta = 1024;  // nonzeros per pass

template <int J>
__global__ void k_gather_bf16_fh(float* out, const uint32_t* meta_g, int passes) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* meta = reinterpret_cast<uint32_t*>(sm + kWinBytes);
  for (int i = threadIdx.x; i < kWinBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u ^ i;
  for (int i = threadIdx.x; i < kMeta; i += blockDim.x) meta[i] = meta_g[i];
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + (threadIdx.x & 31) * 16 +
                        ((threadIdx.x >> 5) & 3) * 512;
  float acc[J][8];
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[j][i] = 0.f;
  const long long t0 = clock64();
  for (int p = 0; p < passes; ++p) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint4* mq = reinterpret_cast<const uint4*>(meta + j * (kMeta / J));
#pragma unroll 2
      for (int q = 0; q < kMeta / J / 4; ++q) {
        const uint4 m4 = mq[q];
        const uint32_t mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t addr = base + (mm[u] >> 16);
          uint32_t v0, v1, v2, v3;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(addr));
          const uint32_t vv[4] = {v0, v1, v2, v3};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            asm("{\n\t.reg .b16 l, h, wl, wh;\n\tmov.b32 {l,h}, %2;\n\tmov.b32 {wl,wh}, %3;\n\t"
                "fma.rn.f32.bf16 %0, l, wl, %0;\n\t"
                "fma.rn.f32.bf16 %1, h, wl, %1;\n\t}"
                : "+f"(acc[j][2 * k]), "+f"(acc[j][2 * k + 1])
                : "r"(vv[k]), "r"(mm[u]));
          }
        }
      }
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// unpack bf16 -> f32 with PRMT/shift, then scalar FFMA with an fp32 weight
template <int J>
__global__ void k_gather_bf16_unpack(float* out, const uint32_t* meta_g, const float* wv_g, int passes) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* meta = reinterpret_cast<uint32_t*>(sm + kWinBytes);
  float* wv = reinterpret_cast<float*>(sm + kWinBytes + kMeta * 4);
  for (int i = threadIdx.x; i < kWinBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u ^ i;
  for (int i = threadIdx.x; i < kMeta; i += blockDim.x) {
    meta[i] = meta_g[i];
    wv[i] = wv_g[i];
  }
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + (threadIdx.x & 31) * 16 +
                        ((threadIdx.x >> 5) & 3) * 512;
  float acc[J][8];
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[j][i] = 0.f;
  const long long t0 = clock64();
  for (int p = 0; p < passes; ++p) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint4* mq = reinterpret_cast<const uint4*>(meta + j * (kMeta / J));
      const float4* wq = reinterpret_cast<const float4*>(wv + j * (kMeta / J));
#pragma unroll 2
      for (int q = 0; q < kMeta / J / 4; ++q) {
        const uint4 m4 = mq[q];
        const float4 w4 = wq[q];
        const uint32_t mm[4] = {m4.x, m4.y, m4.z, m4.w};
        const float ww[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t addr = base + (mm[u] >> 16);
          uint32_t v0, v1, v2, v3;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(addr));
          const uint32_t vv[4] = {v0, v1, v2, v3};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc[j][2 * k] = fmaf(ww[u], __uint_as_float(vv[k] << 16), acc[j][2 * k]);
            acc[j][2 * k + 1] = fmaf(ww[u], __uint_as_float(vv[k] & 0xFFFF0000u), acc[j][2 * k + 1]);
          }
        }
      }
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// fp32 window: 4 images per 16-byte vector, fma.rn.f32x2 with the weight pair
template <int J>
__global__ void k_gather_f32_ffma2(float* out, const uint32_t* meta_g, const float* wv_g, int passes) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* meta = reinterpret_cast<uint32_t*>(sm + kWinBytes);
  float* wv = reinterpret_cast<float*>(sm + kWinBytes + kMeta * 4);
  for (int i = threadIdx.x; i < kWinBytes / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f + i * 1e-6f;
  for (int i = threadIdx.x; i < kMeta; i += blockDim.x) {
    meta[i] = meta_g[i];
    wv[i] = wv_g[i];
  }
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + (threadIdx.x & 31) * 16 +
                        ((threadIdx.x >> 5) & 3) * 512;
  unsigned long long acc[J][2];
#pragma unroll
  for (int j = 0; j < J; ++j) acc[j][0] = acc[j][1] = 0ull;
  const long long t0 = clock64();
  for (int p = 0; p < passes; ++p) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint4* mq = reinterpret_cast<const uint4*>(meta + j * (kMeta / J));
      const float4* wq = reinterpret_cast<const float4*>(wv + j * (kMeta / J));
#pragma unroll 2
      for (int q = 0; q < kMeta / J / 4; ++q) {
        const uint4 m4 = mq[q];
        const float4 w4 = wq[q];
        const uint32_t mm[4] = {m4.x, m4.y, m4.z, m4.w};
        const float ww[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t addr = base + (mm[u] >> 16);
          unsigned long long x01, x23;
          asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(x01), "=l"(x23) : "r"(addr));
          float2 wp = make_float2(ww[u], ww[u]);
          unsigned long long w2 = *reinterpret_cast<unsigned long long*>(&wp);
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j][0]) : "l"(x01), "l"(w2));
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j][1]) : "l"(x23), "l"(w2));
        }
      }
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    float2 a = *reinterpret_cast<float2*>(&acc[j][0]);
    float2 b = *reinterpret_cast<float2*>(&acc[j][1]);
    s += a.x + a.y + b.x + b.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

template <typename F>
int run(const char* name, F launch, int blocks, int threads, double macs_per_thread, int blocks_per_sm) {
  std::vector<unsigned long long> cyc(blocks);
  launch();  // warm
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  CK(cudaMemcpyFromSymbol(cyc.data(), g_cycles, sizeof(unsigned long long) * blocks));
  double mx = 0, sum = 0;
  for (auto c : cyc) {
    mx = c > mx ? c : mx;
    sum += c;
  }
  const double avg = sum / blocks;
  const double per_sm = macs_per_thread * threads * blocks_per_sm / avg;
  printf("%-28s MAC/clk/SM = %7.1f   (avg cyc %.0f, max %.0f, %.3f ms, %.1f TMAC/s wall)\n", name, per_sm, avg, mx,
         ms, macs_per_thread * threads * blocks / (ms * 1e-3) / 1e12);
  return 0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  CK(cudaMalloc(&out, 1 << 24));
  const int iters = 4096;
  printf("SMs %d\n", nsm);
  for (int tpb : {256, 512, 1024}) {
    const int blocks = nsm * (2048 / tpb);
    printf("-- %d threads/block, %d blocks/SM\n", tpb, 2048 / tpb);
    run("ffma (3-reg)", [&] { k_ffma<<<blocks, tpb>>>(out, 1.0001f, iters); }, blocks, tpb, 16.0 * iters, 2048 / tpb);
    run("ffma2 (f32x2)", [&] { k_ffma2<<<blocks, tpb>>>(out, 1.0001f, iters); }, blocks, tpb, 16.0 * iters, 2048 / tpb);
    run("fhfma.bf16 (mixed)", [&] { k_fhfma<<<blocks, tpb>>>(out, 1.0001f, iters); }, blocks, tpb, 16.0 * iters, 2048 / tpb);
  }
  // metadata: random offsets into the window (16-byte aligned, < 64 KB + lane span)
  std::vector<uint32_t> meta(kMeta);
  std::vector<float> wv(kMeta);
  uint32_t s = 12345;
  for (int i = 0; i < kMeta; ++i) {
    s = s * 1664525u + 1013904223u;
    const uint32_t off = ((s >> 8) % (60 * 1024 / 16)) * 16;
    __nv_bfloat16 b = __float2bfloat16(0.01f * (i % 7));
    meta[i] = (off << 16) | *reinterpret_cast<uint16_t*>(&b);
    wv[i] = 0.01f * (i % 7);
  }
  uint32_t* meta_d;
  float* wv_d;
  CK(cudaMalloc(&meta_d, kMeta * 4));
  CK(cudaMalloc(&wv_d, kMeta * 4));
  CK(cudaMemcpy(meta_d, meta.data(), kMeta * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(wv_d, wv.data(), kMeta * 4, cudaMemcpyHostToDevice));
  const int smem = kWinBytes + kMeta * 8;
  CK(cudaFuncSetAttribute(k_gather_bf16_fh<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_gather_bf16_fh<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_gather_bf16_unpack<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_gather_f32_ffma2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int passes = 16;
  for (int tpb : {256, 384, 512, 768}) {
    const int blocks = nsm;
    printf("-- gather loops, %d threads/block, 1 block/SM\n", tpb);
    run("lds128 bf16x8 fhfma J8", [&] { k_gather_bf16_fh<8><<<blocks, tpb, smem>>>(out, meta_d, passes); }, blocks, tpb,
        8.0 * kMeta * passes, 1);
    run("lds128 bf16x8 fhfma J4", [&] { k_gather_bf16_fh<4><<<blocks, tpb, smem>>>(out, meta_d, passes); }, blocks, tpb,
        8.0 * kMeta * passes, 1);
    run("lds128 bf16x8 unpack+ffma J8",
        [&] { k_gather_bf16_unpack<8><<<blocks, tpb, smem>>>(out, meta_d, wv_d, passes); }, blocks, tpb,
        8.0 * kMeta * passes, 1);
    run("lds128 f32x4 ffma2 J8", [&] { k_gather_f32_ffma2<8><<<blocks, tpb, smem>>>(out, meta_d, wv_d, passes); },
        blocks, tpb, 4.0 * kMeta * passes, 1);
  }
  CK(cudaGetLastError());
  return 0;
}
