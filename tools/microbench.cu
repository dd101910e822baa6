// Microbenchmarks that decide the softmax design of the fused attention
// kernel on B200: MUFU ex2 throughput for f32 / f16x2 / bf16x2, and TMEM
// load throughput (tcgen05.ld 32x32b.x32) per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kIters = 4096;

template <int MODE>
__global__ void ex2_kernel(float* out, long long* clk) {
  uint32_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u + threadIdx.x + i;   // f16x2 (1,1)-ish
  float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      } else if (MODE == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
      } else {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += f[i] + __uint_as_float(v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void tmem_ld_kernel(float* out, long long* clk, int nwarps_active) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = base + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < nwarps_active) {
    for (int it = 0; it < kIters / 16; ++it) {
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
            "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
            "=r"(r[31])
          : "r"(tm + (it & 3) * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= r[i];
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}


__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pk(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}
// softmax exp-phase pattern: per iteration 128 keys per thread (4 pieces of
// 32): [ld S piece] -> 32 x (FFMA + MUFU) -> 16 F2FP -> st P piece
template <int MODE>
__global__ void exp_phase_kernel(float* out, long long* clk, int active_warps) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = base + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 256;
  float acc = 0.f;
  const float sl2 = 0.25f, nb = -1.f;
  long long t0 = clock64();
  if (warp < active_warps) {
    uint32_t sa[32];
    if (MODE != 0) { ld32(tm, sa); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
    else {
#pragma unroll
      for (int j = 0; j < 32; ++j) sa[j] = __float_as_uint(-0.01f * j);
    }
    for (int it = 0; it < 64; ++it) {
#pragma unroll 1
      for (int pc = 0; pc < 4; ++pc) {
        if (MODE == 2) { ld32(tm + 32 * pc, sa); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          w[j] = pk(ex2f(fmaf(__uint_as_float(sa[2 * j]), sl2, nb)),
                    ex2f(fmaf(__uint_as_float(sa[2 * j + 1]), sl2, nb)));
        if (MODE >= 1) st16(tm + 128 + 16 * pc, w);
        else {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc += __uint_as_float(w[j]);
        }
      }
    }
    if (MODE >= 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

// XU-pipe sharing: ex2 alone, ex2 + F2FP bf16x2 pack (1 per 2 ex2), ex2 + PRMT pack
template <int MODE>
__global__ void xu_kernel(float* out, long long* clk) {
  float f[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = -0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
    if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t w;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w) : "f"(f[2 * i]), "f"(f[2 * i + 1]));
        acc ^= w;
      }
    } else if (MODE == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t w;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(w) : "r"(__float_as_uint(f[2 * i])),
                     "r"(__float_as_uint(f[2 * i + 1])));
        acc ^= w;
      }
    } else if (MODE == 3) {   // pack only (no ex2 dependence chain change)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t w;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w) : "f"(f[2 * i]), "f"(f[2 * i + 1]));
        acc ^= w;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float a = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) a += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + (float)acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// Full per-pair softmax work, register-resident: MODE 0 = 2 FFMA + 2 ex2.f32 +
// cvt.rn.bf16x2 (the kernel today); MODE 1 = 2 FFMA + cvt.rn.f16x2.f32 +
// ex2.approx.f16x2 (P as packed f16); MODE 2 = MODE 1 with ex2.approx.ftz.bf16x2
// on a bf16x2 argument (not accurate enough; throughput reference only).
template <int MODE>
__global__ void pair_kernel(float* out, long long* clk) {
  float s[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) s[j] = -0.01f * (threadIdx.x + j);
  const float sl2 = 0.25f;
  float nb = -1.f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters / 8; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float a = fmaf(s[2 * j], sl2, nb), b = fmaf(s[2 * j + 1], sl2, nb);
      uint32_t w;
      if (MODE == 0) {
        float ea, eb;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(ea) : "f"(a));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(eb) : "f"(b));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w) : "f"(eb), "f"(ea));
      } else if (MODE == 1) {
        uint32_t h;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(w) : "r"(h));
      } else {
        uint32_t h;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(w) : "r"(h));
      }
      acc += w;
    }
    nb -= 1e-7f;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&clk, 148 * sizeof(long long));
  long long h[148];
  const char* names[3] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2"};
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) ex2_kernel<0><<<148, 32 * warps>>>(out, clk);
        if (mode == 1) ex2_kernel<1><<<148, 32 * warps>>>(out, clk);
        if (mode == 2) ex2_kernel<2><<<148, 32 * warps>>>(out, clk);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
      double ops = (double)kIters * 8 * 32 * warps;   // lane-ops per SM
      printf("%-22s warps/SM %2d: %.2f lane-ops/clk/SM (%lld clk)\n", names[mode], warps,
             ops / h[0], h[0]);
    }
  }
  for (int w = 1; w <= 16; w *= 2) {
    for (int rep = 0; rep < 2; ++rep) tmem_ld_kernel<<<148, 512>>>(out, clk, w);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("tmem kernel failed: %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = (double)(kIters / 16) * 32 * 32 * 4 * w;
    printf("tcgen05.ld x32, %2d warps: %.1f B/clk/SM (%lld clk)\n", w, bytes / h[0], h[0]);
  }
  {
    const char* xn[3] = {"ex2 only", "ex2 + cvt.bf16x2 (1 per 2)", "ex2 + prmt (1 per 2)"};
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) xu_kernel<0><<<148, 256>>>(out, clk);
        if (mode == 1) xu_kernel<1><<<148, 256>>>(out, clk);
        if (mode == 2) xu_kernel<2><<<148, 256>>>(out, clk);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
      double ex = (double)(kIters / 4) * 16 * 256;
      printf("%-28s: %.2f ex2/clk/SM\n", xn[mode], ex / h[0]);
    }
  }
  const char* en[3] = {"regs only", "+st P", "+ld S +st P"};
  for (int mode = 0; mode < 3; ++mode)
    for (int w = 4; w <= 8; w += 4) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) exp_phase_kernel<0><<<148, 256>>>(out, clk, w);
        if (mode == 1) exp_phase_kernel<1><<<148, 256>>>(out, clk, w);
        if (mode == 2) exp_phase_kernel<2><<<148, 256>>>(out, clk, w);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("exp_phase failed: %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
      double elems = 64.0 * 128 * 32 * w;
      printf("exp phase %-12s warps %d: %.2f exp/clk/SM (%.0f clk per 128x128-per-warp-group chunk-equivalent)\n",
             en[mode], w, elems / h[0], (double)h[0] / 64);
    }
  {
    const char* pn[3] = {"f32: 2 FFMA+2 MUFU+F2FP", "f16x2: 2 FFMA+F2FP+MUFU.f16x2",
                         "bf16x2: 2 FFMA+F2FP+MUFU.bf16x2"};
    for (int warps = 4; warps <= 16; warps *= 2)
      for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
          if (mode == 0) pair_kernel<0><<<148, 32 * warps>>>(out, clk);
          if (mode == 1) pair_kernel<1><<<148, 32 * warps>>>(out, clk);
          if (mode == 2) pair_kernel<2><<<148, 32 * warps>>>(out, clk);
        }
        cudaDeviceSynchronize();
        cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
        double ex = (double)(kIters / 8) * 32 * 32 * warps;
        printf("pair %-34s warps %2d: %.2f exp/clk/SM\n", pn[mode], warps, ex / h[0]);
      }
  }
  return 0;
}
