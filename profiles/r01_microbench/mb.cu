// Microbenchmarks to inform the design: streaming read BW and warp-aggregation cost.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

struct __align__(16) Rec { uint64_t count, seq; uint32_t comm; uint16_t nr, rank, dev, aux, aux2; uint8_t kc, ad; };

__global__ void k_read(const int4* __restrict__ p, size_t n16, unsigned long long* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (; i < n16; i += st) { int4 v = __ldg(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345) atomicAdd(out, 1ull);
}
// records: one thread per record, two 16B loads
__global__ void k_rec(const Rec* __restrict__ p, size_t n, unsigned long long* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (; i < n; i += st) { const int4* q = (const int4*)(p + i); int4 a = __ldg(q), b = __ldg(q + 1); acc ^= a.x ^ b.w ^ a.z; }
  if (acc == 0x12345) atomicAdd(out, 1ull);
}
// warp aggregation: key = rank (i & 7) etc; match_any + redux 16-bit chunks, then smem atomics
template <int MODE>
__global__ void k_agg(const Rec* __restrict__ p, size_t n, unsigned long long* out) {
  __shared__ unsigned long long hb[1024]; __shared__ unsigned hf[1024];
  for (int j = threadIdx.x; j < 1024; j += blockDim.x) { hb[j] = 0; hf[j] = 0; }
  __syncthreads();
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  int lane = threadIdx.x & 31;
  for (; i < n + 0; i += st) {
    const int4* q = (const int4*)(p + i); int4 a = __ldg(q), b = __ldg(q + 1);
    unsigned key = ((unsigned)b.y >> 16) & 1023;   // rank field
    unsigned long long v = ((unsigned long long)(unsigned)a.y << 32) | (unsigned)a.x;
    if (MODE == 0) { atomicAdd(&hb[key], v); atomicAdd(&hf[key], 1u); }
    else {
      unsigned m = __match_any_sync(0xffffffffu, key);
      unsigned c0 = __reduce_add_sync(m, (unsigned)(v & 0xffff));
      unsigned c1 = __reduce_add_sync(m, (unsigned)((v >> 16) & 0xffff));
      unsigned c2 = __reduce_add_sync(m, (unsigned)((v >> 32) & 0xffff));
      unsigned c3 = __reduce_add_sync(m, (unsigned)(v >> 48));
      if (lane == __ffs(m) - 1) {
        unsigned long long s = (unsigned long long)c0 + ((unsigned long long)c1 << 16) + ((unsigned long long)c2 << 32) + ((unsigned long long)c3 << 48);
        atomicAdd(&hb[key], s); atomicAdd(&hf[key], (unsigned)__popc(m));
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 1024; j += blockDim.x) if (hf[j]) { atomicAdd(out, hb[j]); atomicAdd(out + 1, (unsigned long long)hf[j]); }
}
__global__ void k_fill(Rec* p, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) { Rec r{}; r.count = (i * 2654435761ull) & 0xfffffff; r.seq = i / 8; r.rank = i & 7; r.nr = 8; r.dev = i & 7; p[i] = r; }
}
int main() {
  size_t n = 1ull << 28; // 268M records = 8.6 GB
  Rec* d; CK(cudaMalloc(&d, n * sizeof(Rec)));
  unsigned long long* o; CK(cudaMalloc(&o, 64)); CK(cudaMemset(o, 0, 64));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k_fill<<<sms * 8, 256>>>(d, n); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto fn) {
    for (int w = 0; w < 2; w++) fn();
    cudaEventRecord(e0); for (int r = 0; r < 5; r++) fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-28s %8.3f ms  %8.1f GB/s  %8.2f Grec/s\n", name, ms, n * 32.0 / ms / 1e6, n / ms / 1e6);
  };
  for (int bpsm : {4, 8, 16}) {
    char nm[64];
    sprintf(nm, "read int4 bpsm=%d", bpsm); run(nm, [&]{ k_read<<<sms * bpsm, 256>>>((const int4*)d, n * 2, o); });
    sprintf(nm, "rec 2xint4 bpsm=%d", bpsm); run(nm, [&]{ k_rec<<<sms * bpsm, 256>>>(d, n, o); });
    sprintf(nm, "agg atomics bpsm=%d", bpsm); run(nm, [&]{ k_agg<0><<<sms * bpsm, 256>>>(d, n, o); });
    sprintf(nm, "agg match+redux bpsm=%d", bpsm); run(nm, [&]{ k_agg<1><<<sms * bpsm, 256>>>(d, n, o); });
  }
  CK(cudaGetLastError());
  return 0;
}
