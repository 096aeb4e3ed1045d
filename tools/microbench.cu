// Microbenchmarks for the B200 memory system: the primitive access patterns
// the BOBA pipeline is built from (coalesced streaming, random 4-byte gather
// from an L2-sized table, random RED.MIN / RED.ADD, guarded atomics).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hash32(uint32_t x){ x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }

__global__ void k_fill_idx(uint32_t* idx, size_t n, uint32_t tbl, int skew){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for (; i<n; i+= (size_t)gridDim.x*blockDim.x){
    uint32_t h = hash32((uint32_t)i*2654435761u + 12345u);
    if (skew){ // crude power law: square of a uniform in [0,1) mapped then scrambled
      double u = (h & 0xFFFFFF) / 16777216.0; u = u*u*u; uint32_t v = (uint32_t)(u * tbl);
      idx[i] = hash32(v ^ 0x9e3779b9u) % tbl;  // scatter hot ids randomly
    } else idx[i] = h % tbl;
  }
}
__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for (; i<n; i+= (size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
__global__ void k_read(const int4* __restrict__ a, size_t n, int* sink){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; int acc=0;
  for (; i<n; i+= (size_t)gridDim.x*blockDim.x){ int4 v=a[i]; acc ^= v.x^v.y^v.z^v.w; }
  if (acc==0x12345678) *sink=acc;
}
__global__ void k_gather(const uint4* __restrict__ idx, const uint32_t* __restrict__ tbl, uint4* __restrict__ out, size_t n4){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for (; i<n4; i+= (size_t)gridDim.x*blockDim.x){ uint4 v=idx[i]; uint4 r; r.x=__ldg(tbl+v.x); r.y=__ldg(tbl+v.y); r.z=__ldg(tbl+v.z); r.w=__ldg(tbl+v.w); out[i]=r; }
}
__global__ void k_redmin(const uint4* __restrict__ idx, uint32_t* tbl, size_t n4){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for (; i<n4; i+= (size_t)gridDim.x*blockDim.x){ uint4 v=idx[i]; uint32_t p=(uint32_t)i*4; atomicMin(tbl+v.x,p); atomicMin(tbl+v.y,p+1); atomicMin(tbl+v.z,p+2); atomicMin(tbl+v.w,p+3);} }
__global__ void k_guardmin(const uint4* __restrict__ idx, uint32_t* tbl, size_t n4){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for (; i<n4; i+= (size_t)gridDim.x*blockDim.x){ uint4 v=idx[i]; uint32_t p=(uint32_t)i*4;
    uint32_t a=tbl[v.x], b=tbl[v.y], c=tbl[v.z], d=tbl[v.w];
    if (p<a) atomicMin(tbl+v.x,p); if (p+1<b) atomicMin(tbl+v.y,p+1); if (p+2<c) atomicMin(tbl+v.z,p+2); if (p+3<d) atomicMin(tbl+v.w,p+3);} }
__global__ void k_redadd(const uint4* __restrict__ idx, uint32_t* tbl, size_t n4){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for (; i<n4; i+= (size_t)gridDim.x*blockDim.x){ uint4 v=idx[i]; atomicAdd(tbl+v.x,1); atomicAdd(tbl+v.y,1); atomicAdd(tbl+v.z,1); atomicAdd(tbl+v.w,1);} }
__global__ void k_scatter(const uint4* __restrict__ idx, uint32_t* tbl, size_t n4){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for (; i<n4; i+= (size_t)gridDim.x*blockDim.x){ uint4 v=idx[i]; tbl[v.x]=i; tbl[v.y]=i; tbl[v.z]=i; tbl[v.w]=i;} }

int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,dev));
  printf("%s SMs=%d L2=%d MB persistL2max=%d MB\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize>>20, pr.persistingL2CacheMaxSize>>20);
  const size_t N = 1ull<<27; // 134M accesses (= 2m at R-MAT s22 ef16)
  uint32_t *idx, *tbl, *out; int* sink;
  CK(cudaMalloc(&idx, N*4)); CK(cudaMalloc(&out, N*4)); CK(cudaMalloc(&tbl, (size_t)1<<30)); CK(cudaMalloc(&sink,4));
  void* big; size_t BIG = 2ull<<30; CK(cudaMalloc(&big, 2*BIG));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int G = pr.multiProcessorCount*8, B=256;
  auto T = [&](auto fn, int reps)->float{ fn(); cudaDeviceSynchronize(); float best=1e9; for(int r=0;r<reps;r++){ cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;} return best; };
  float t = T([&]{ k_copy<<<G,B>>>((int4*)big, (int4*)((char*)big+BIG), BIG/16); }, 5);
  printf("copy 2GiB: %.3f ms  %.1f GB/s (r+w)\n", t, 2.0*BIG/t/1e6);
  t = T([&]{ k_read<<<G,B>>>((int4*)big, BIG/16, sink); }, 5);
  printf("read 2GiB: %.3f ms  %.1f GB/s\n", t, 1.0*BIG/t/1e6);
  for (int skew=0; skew<2; skew++)
  for (uint32_t mb : {4u, 16u, 64u, 128u, 256u, 1024u}){
    uint32_t tn = mb*(1u<<20)/4;
    k_fill_idx<<<G,B>>>(idx, N, tn, skew); CK(cudaDeviceSynchronize());
    float tg = T([&]{ k_gather<<<G,B>>>((uint4*)idx, tbl, (uint4*)out, N/4); }, 5);
    float tm = T([&]{ cudaMemsetAsync(tbl, 0xFF, (size_t)tn*4); k_redmin<<<G,B>>>((uint4*)idx, tbl, N/4); }, 5);
    float tgm = T([&]{ cudaMemsetAsync(tbl, 0xFF, (size_t)tn*4); k_guardmin<<<G,B>>>((uint4*)idx, tbl, N/4); }, 5);
    float tms = T([&]{ cudaMemsetAsync(tbl, 0xFF, (size_t)tn*4); }, 5);
    float ta = T([&]{ k_redadd<<<G,B>>>((uint4*)idx, tbl, N/4); }, 5);
    float ts = T([&]{ k_scatter<<<G,B>>>((uint4*)idx, tbl, N/4); }, 5);
    printf("skew=%d table %4u MB: gather %.3f ms (%.1f G/s) | redmin %.3f (%.1f G/s) | guardmin %.3f | memset %.3f | redadd %.3f (%.1f G/s) | scatter %.3f\n",
      skew, mb, tg, N/tg/1e6, tm-tms, N/(tm-tms)/1e6, tgm-tms, tms, ta, N/ta/1e6, ts);
  }
  return 0;
}
