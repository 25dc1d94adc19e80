// Probe for the MN-major SWIZZLE_128B tf32 UMMA operand encoding (debug tool, not product code).
// A[m][k] (m < 128, k < 8) written by hand in the canonical swizzled MN-major layout,
// D = A A^T by one tcgen05.mma kind::tf32, compared with the host product.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void probe(float *out, uint32_t idesc, uint32_t lbo, uint32_t sbo, uint32_t ltype, uint32_t blk, int var) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4 * (int)blk / 4; i += blockDim.x) ((float *)sm)[i] = 0.f;
  __syncthreads();
  for (int e = threadIdx.x; e < 128 * 8; e += blockDim.x) {
    int m = e / 8, k = e % 8;
    float v = (float)((m * 7 + k * 3) % 11) - 5.0f;
    int b = m / 32, mm = m % 32, chunk = mm / 4;
    uint32_t off;
    if (var == 0) off = b * blk + k * 128 + ((chunk ^ (k & 7)) * 16) + (mm % 4) * 4;          // 16B chunks ^ row%8
    else if (var == 1) off = b * blk + k * 128 + ((((mm / 8) ^ (k & 3)) * 32)) + (mm % 8) * 4;  // 32B chunks ^ row%4
    else off = b * blk + k * 128 + ((((mm / 8) ^ ((k >> 1) & 3)) * 32)) + (mm % 8) * 4;        // 32B chunks ^ (row/2)%4
    *(float *)(sm + off) = v;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    uint64_t d = 0;
    uint32_t sa = smem_u32(sm);
    d |= (uint64_t)((sa >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)ltype << 61;
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 0;\n" ::"r"(tmem), "l"(d), "l"(d), "r"(idesc) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncwarp();
  if (w < 4) {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    for (int cb = 0; cb < 4; ++cb) {
      uint32_t r[32];
      uint32_t taddr = tmem + ((uint32_t)(w * 32) << 16) + (uint32_t)(cb * 32);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int q = 0; q < 32; ++q) out[(w * 32 + lane) * 128 + cb * 32 + q] = __uint_as_float(r[q]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tmem) : "memory");
}
int main() {
  float *d_out; cudaMalloc(&d_out, 128 * 128 * 4);
  static float h[128 * 128]; float A[128][8];
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) A[m][k] = (float)((m * 7 + k * 3) % 11) - 5.0f;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const uint32_t base = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t idesc = base | (1u << 15) | (1u << 16);
  const uint32_t blk = 4096;
  for (int var = 0; var < 3; ++var)
  for (uint32_t lt : {1u, 2u})
  for (uint32_t sbo : {512u, 1024u, 128u}) {
    uint32_t lbo = blk;
    cudaMemset(d_out, 0, 128 * 128 * 4);
    probe<<<1, 128, 48 * 1024>>>(d_out, idesc, lbo, sbo, lt, blk, var);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("var %d lt %u sbo %u: error %s\n", var, lt, sbo, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    double err = 0, nz = 0;
    for (int i = 0; i < 128; ++i) for (int j = 0; j < 128; ++j) {
      double ref = 0; for (int k = 0; k < 8; ++k) ref += (double)A[i][k] * A[j][k];
      err = fmax(err, fabs(h[i * 128 + j] - ref)); nz += fabs(h[i * 128 + j]);
    }
    printf("var %d ltype %u lbo %u sbo %u: max err %.3g (sum|D| %.3g)\n", var, lt, lbo, sbo, err, nz);
  }
  return 0;
}
