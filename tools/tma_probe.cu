// Standalone TMA legality probe: one CTA loads one box into smem and reports the bytes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__global__ void probe(const __grid_constant__ CUtensorMap map, int rank, int c0, unsigned bytes, unsigned char* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* dst = (unsigned char*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), d = (uint32_t)__cvta_generic_to_shared(dst);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bytes));
    if (rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   :: "r"(d), "l"(&map), "r"(b), "r"(c0), "r"(0) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   :: "r"(d), "l"(&map), "r"(b), "r"(c0), "r"(0), "r"(0) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(b));
    for (int i = 0; i < 64; ++i) out[i] = dst[i];
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int rank = atoi(argv[1]), bx0 = atoi(argv[2]), bx1 = atoi(argv[3]), bx2 = atoi(argv[4]), sw = atoi(argv[5]);
  int c0 = argc > 6 ? atoi(argv[6]) : 0;
  long T = 2432, L = 64;
  unsigned char *g, *out;
  cudaMalloc(&g, 3 * T * L); cudaMalloc(&out, 64);
  cudaMemset(g, 7, 3 * T * L);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)T, (cuuint64_t)L, 3}, str[2] = {(cuuint64_t)T, (cuuint64_t)(T * L)};
  cuuint32_t box[3] = {(cuuint32_t)bx0, (cuuint32_t)bx1, (cuuint32_t)bx2}, es[3] = {1, 1, 1};
  CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned bytes = bx0 * bx1 * (rank == 3 ? bx2 : 1);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  probe<<<1, 32, 100000>>>(m, rank, c0, bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned char h[64]; cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
  printf("rank %d box %d %d %d sw %d c0 %d: encode %d run %s first %d\n", rank, bx0, bx1, bx2, sw, c0, (int)rc, cudaGetErrorString(e), h[0]);
  return 0;
}
