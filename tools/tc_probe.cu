// Probe of the sm_100a primitives the tcgen05 decode-attention kernel relies on
// (run once on a B200; prints PASS/FAIL lines):
//   1. tcgen05.st.16x128b / 16x256b thread -> (lane, column) mapping
//   2. kind::i8 MMA, A (u8) from TMEM, B (s8) from smem MN-major, D s32, M=128, N=16/32
//   3. kind::i8 MMA, A (u8) from smem K-major (no swizzle), B (u8) MN-major
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void st16x128(uint32_t ta, uint32_t r0, uint32_t r1) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x1.b32 [%0], {%1, %2};" ::"r"(ta), "r"(r0), "r"(r1));
}
__device__ __forceinline__ void st16x256(uint32_t ta, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta), "r"(r0), "r"(r1), "r"(r2),
               "r"(r3));
}
__device__ __forceinline__ void st32x32x8(uint32_t ta, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
__device__ __forceinline__ void ld32x32x8(uint32_t ta, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint64_t desc_none(const void* base, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(base) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  return d;                // layout 0 = SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_signed, int b_signed, int a_mn, int b_mn) {
  return (2u << 4) | ((uint32_t)a_signed << 7) | ((uint32_t)b_signed << 10) | ((uint32_t)a_mn << 15) |
         ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// out layout: [0..127] 16x128b map, [128..255] 16x256b map (value = 1000*thread + reg, read back
// as lane*8+col for lanes 0..15, cols 0..7); then MMA results
__global__ void probe(const uint8_t* A, const int8_t* B, const uint8_t* A2, const uint8_t* B2, int* out) {
  __shared__ uint32_t taddr_s;
  __shared__ __align__(128) uint8_t sB[128 * 32];   // MN-major [k][32 bytes] as 2 n-groups of 16
  __shared__ __align__(128) uint8_t sA[128 * 32];   // K-major A2 (M=128 x K=32)
  __shared__ __align__(128) uint8_t sB2[32 * 16];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;
  // ---- 1. store-shape mapping (warp 0, lanes 0..15, columns 0..7) ----
  if (warp == 0) {
    st16x128(T + 0, 1000 * lane + 0, 1000 * lane + 1);
    st16x256(T + 8, 1000 * lane + 0, 1000 * lane + 1, 1000 * lane + 2, 1000 * lane + 3);
    st_wait();
    uint32_t v[8];
    ld32x32x8(T + 0, v);
    if (lane < 16)
      for (int c = 0; c < 8; ++c) out[lane * 8 + c] = (int)v[c];
    ld32x32x8(T + 8, v);
    if (lane < 16)
      for (int c = 0; c < 8; ++c) out[128 + lane * 8 + c] = (int)v[c];
  }
  // ---- 2. A (u8 [128][32]) into TMEM cols 16..23 (thread = row), B s8 [32 k][32 n] MN-major ----
  {
    uint32_t w[8];
    for (int i = 0; i < 8; ++i) w[i] = reinterpret_cast<const uint32_t*>(A + tid * 32)[i];
    st32x32x8(T + ((uint32_t)(32 * warp) << 16) + 16, w);
    st_wait();
  }
  // MN-major no-swizzle: n-group (16 bytes of N) g at g*SBO, k row at 16*k within a core
  // matrix of 8 rows, k-groups at LBO = 128
  for (int i = tid; i < 32 * 32; i += 128) {
    const int k = i / 32, n = i % 32;
    sB[(n / 16) * 512 + k * 16 + (n % 16)] = (uint8_t)B[k * 32 + n];
  }
  // K-major no-swizzle A2 [128 m][32 k]: core matrix (8 rows x 16 B) contiguous; m-groups at SBO=128,
  // k-chunks (16 B) at LBO = 128*16 = 2048
  for (int i = tid; i < 128 * 32; i += 128) {
    const int m = i / 32, k = i % 32;
    sA[(k / 16) * 2048 + m * 16 + (k % 16)] = A2[i];
  }
  for (int i = tid; i < 32 * 16; i += 128) {
    const int k = i / 16, n = i % 16;
    sB2[k * 16 + n] = B2[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    // N = 32, u8 x s8 -> cols 64..95
    mma_i8_ts(T + 64, T + 16, desc_none(sB, 128, 512), idesc_i8(128, 32, 0, 1, 0, 1), 0);
    // N = 16 (first n-group) -> cols 96..111
    mma_i8_ts(T + 96, T + 16, desc_none(sB, 128, 512), idesc_i8(128, 16, 0, 1, 0, 1), 0);
    // SS: A2 K-major u8, B2 MN-major u8, N = 16 -> cols 128..143
    mma_i8_ss(T + 128, desc_none(sA, 2048, 128), desc_none(sB2, 128, 256), idesc_i8(128, 16, 0, 0, 0, 1), 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  {
    uint32_t v[8];
    const uint32_t lb = (uint32_t)(32 * warp) << 16;
    for (int c0 = 0; c0 < 32; c0 += 8) {
      ld32x32x8(T + lb + 64 + c0, v);
      for (int c = 0; c < 8; ++c) out[256 + tid * 32 + c0 + c] = (int)v[c];
    }
    for (int c0 = 0; c0 < 16; c0 += 8) {
      ld32x32x8(T + lb + 96 + c0, v);
      for (int c = 0; c < 8; ++c) out[256 + 4096 + tid * 16 + c0 + c] = (int)v[c];
      ld32x32x8(T + lb + 128 + c0, v);
      for (int c = 0; c < 8; ++c) out[256 + 4096 + 2048 + tid * 16 + c0 + c] = (int)v[c];
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(T));
}

int main() {
  std::vector<uint8_t> A(128 * 32), A2(128 * 32), B2(32 * 16);
  std::vector<int8_t> B(32 * 32);
  srand(1);
  for (auto& x : A) x = rand() & 255;
  for (auto& x : A2) x = rand() & 255;
  for (auto& x : B) x = (int8_t)(rand() & 255);
  for (auto& x : B2) x = rand() & 255;
  uint8_t *dA, *dA2, *dB2;
  int8_t* dB;
  int* dout;
  const int NOUT = 256 + 4096 + 2048 + 2048;
  cudaMalloc(&dA, A.size()); cudaMalloc(&dA2, A2.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dB2, B2.size());
  cudaMalloc(&dout, NOUT * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dA2, A2.data(), A2.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB2, B2.data(), B2.size(), cudaMemcpyHostToDevice);
  cudaMemset(dout, 0xff, NOUT * 4);
  probe<<<1, 128>>>(dA, dB, dA2, dB2, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<int> out(NOUT);
  cudaMemcpy(out.data(), dout, NOUT * 4, cudaMemcpyDeviceToHost);
  for (int s = 0; s < 2; ++s) {
    printf("%s map (lane: col0..7 = 1000*thread+reg):\n", s ? "16x256b" : "16x128b");
    for (int l = 0; l < 16; ++l) {
      printf("  lane %2d:", l);
      for (int c = 0; c < 8; ++c) printf(" %6d", out[s * 128 + l * 8 + c]);
      printf("\n");
    }
  }
  int bad = 0, bad16 = 0, bad2 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      int ref = 0;
      for (int k = 0; k < 32; ++k) ref += (int)A[m * 32 + k] * (int)B[k * 32 + n];
      if (out[256 + m * 32 + n] != ref) { if (bad < 5) printf("TS N32 m%d n%d got %d want %d\n", m, n, out[256 + m * 32 + n], ref); ++bad; }
      if (n < 16 && out[256 + 4096 + m * 16 + n] != ref) ++bad16;
    }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      int ref = 0;
      for (int k = 0; k < 32; ++k) ref += (int)A2[m * 32 + k] * (int)B2[k * 16 + n];
      if (out[256 + 4096 + 2048 + m * 16 + n] != ref) { if (bad2 < 5) printf("SS m%d n%d got %d want %d\n", m, n, out[256 + 4096 + 2048 + m * 16 + n], ref); ++bad2; }
    }
  printf("i8 TS u8xs8 MN-major B N=32: %s (%d bad)\n", bad ? "FAIL" : "PASS", bad);
  printf("i8 TS u8xs8 MN-major B N=16: %s (%d bad)\n", bad16 ? "FAIL" : "PASS", bad16);
  printf("i8 SS u8xu8 K-major A, MN-major B N=16: %s (%d bad)\n", bad2 ? "FAIL" : "PASS", bad2);
  return 0;
}
