// Recovery remap-table rebuild for sm_100a.
//
// Reference: MemoryModel.vmm_map (pkg/src/mpssim/memory.py:269-283) gives the standby
// one PageRec(GPU, RW, ("alloc", handle)) per 4 KiB page of each shared allocation, i.e.
// standby VA base + i*4096 -> alloc.pages[i]; deploy_pair maps weights and KV this way
// (recovery.py:175-184), and complete_wake restores the live KV block tables
// (recovery.py:342-344; KV block b is KV page b).  Here the table is produced at any
// power-of-two granularity G >= 4 KiB: entry k = (base + k*G, pages[k*G/4096]).
//
// Pure bandwidth: 8 B read + 16 B written per entry.  At G > 4 KiB the read is a stride
// of G/4096 u64, so every read pulls a 64-B L2 fetch for 8 useful bytes.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpsf_kernels.h"

namespace mpsf {

constexpr int RB = 256;
constexpr int REPT = 4;

// One 8-byte page number per entry, G apart: the L2 fetches at least 64 B per miss, and the
// default (a 128-byte fetch) reads twice that -- the 64-byte prefetch size cuts the 64 KiB remap
// from 31 to 23 us (tools/remap_ab.py; profiles/r02/ab_remap.txt).
__device__ __forceinline__ unsigned long long ld_phys(const unsigned long long* p) {
  unsigned long long v;
  asm("ld.global.nc.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(RB) k_remap(uint64_t va_base, const unsigned long long* __restrict__ phys,
                                              uint32_t shift, uint32_t gran_log2, uint64_t E,
                                              ulonglong2* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * RB * REPT;
  for (uint64_t k0 = (uint64_t)blockIdx.x * RB * REPT + threadIdx.x; k0 < E; k0 += stride) {
    unsigned long long p[REPT];
#pragma unroll
    for (int u = 0; u < REPT; ++u) {
      const uint64_t k = k0 + (uint64_t)u * RB;
      p[u] = k < E ? ld_phys(phys + (k << shift)) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < REPT; ++u) {
      const uint64_t k = k0 + (uint64_t)u * RB;
      if (k < E) __stcs(out + k, make_ulonglong2(va_base + (k << gran_log2), p[u]));
    }
  }
}

__global__ void __launch_bounds__(RB) k_remap_blocks(uint64_t va_base, const unsigned long long* __restrict__ phys,
                                                     uint64_t npages, const uint32_t* __restrict__ blocks,
                                                     uint64_t nb, ulonglong2* __restrict__ out,
                                                     uint32_t* __restrict__ err) {
  for (uint64_t j = (uint64_t)blockIdx.x * RB + threadIdx.x; j < nb; j += (uint64_t)gridDim.x * RB) {
    const uint32_t b = __ldcs(blocks + j);
    if (b >= npages) { atomicOr(err, 1u); continue; }
    __stcs(out + j, make_ulonglong2(va_base + ((uint64_t)b << 12), __ldg(phys + b)));
  }
}

static int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int launch_remap(uint64_t va_base, const uint64_t* phys, uint64_t npages4k, uint32_t gran_log2,
                 mpsf_remap_entry* out, cudaStream_t st) {
  const uint32_t shift = gran_log2 - 12;
  const uint64_t step = 1ull << shift;
  const uint64_t E = (npages4k + step - 1) / step;
  if (E == 0) return 0;
  uint64_t blocks = (E + RB * REPT - 1) / (RB * REPT);
  const uint64_t cap = (uint64_t)sms() * 8;
  if (blocks > cap) blocks = cap;
  k_remap<<<(unsigned)blocks, RB, 0, st>>>(va_base, reinterpret_cast<const unsigned long long*>(phys), shift,
                                          gran_log2, E, reinterpret_cast<ulonglong2*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_remap_blocks(uint64_t va_base, const uint64_t* phys, uint64_t npages4k,
                        const uint32_t* blocks, uint64_t nblocks, mpsf_remap_entry* out,
                        uint32_t* err_flag, cudaStream_t st) {
  if (nblocks == 0) return 0;
  uint64_t g = (nblocks + RB - 1) / RB;
  const uint64_t cap = (uint64_t)sms() * 8;
  if (g > cap) g = cap;
  k_remap_blocks<<<(unsigned)g, RB, 0, st>>>(va_base, reinterpret_cast<const unsigned long long*>(phys), npages4k,
                                            blocks, nblocks, reinterpret_cast<ulonglong2*>(out), err_flag);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace mpsf
