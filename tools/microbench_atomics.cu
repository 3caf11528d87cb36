// Secondary-ceiling microbenchmarks: shared-memory and L2/global
// atomic throughput on random addresses. Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t lcg(uint32_t& s){ s = s*1664525u + 1013904223u; return s ^ (s>>16); }

template<int MODE>
__global__ void k_smem(uint32_t* out, int iters, int entries_mask){
  extern __shared__ uint32_t sm[];
  for (int i=threadIdx.x;i<=entries_mask;i+=blockDim.x) sm[i]=0;
  __syncthreads();
  uint32_t s = blockIdx.x*7919u + threadIdx.x*104729u + 1;
  uint32_t acc=0;
  for (int i=0;i<iters;i++){
    uint32_t a = lcg(s) & entries_mask;
    if (MODE==0) atomicAdd(&sm[a],1u);
    else if (MODE==1) acc += atomicAdd(&sm[a],1u);
    else if (MODE==2) { unsigned long long* p=(unsigned long long*)sm; atomicAdd(&p[a>>1],1ull);} 
    else { acc += sm[a]; }
  }
  __syncthreads();
  if (acc==12345) out[0]=acc;
  if (threadIdx.x==0) out[blockIdx.x+1]=sm[threadIdx.x];
}
template<int MODE>
__global__ void k_glob(uint32_t* base, size_t per_cta_mask, int shared_region, int iters){
  uint32_t* row = shared_region ? base : base + (size_t)blockIdx.x*(per_cta_mask+1);
  uint32_t s = blockIdx.x*7919u + threadIdx.x*104729u + 1;
  uint32_t acc=0;
  for (int i=0;i<iters;i++){
    uint32_t a = lcg(s) & per_cta_mask;
    if (MODE==0) atomicAdd(&row[a],1u);
    else if (MODE==1) acc += atomicAdd(&row[a],1u);
    else { unsigned long long* p=(unsigned long long*)row; atomicAdd(&p[a>>1],1ull);} 
  }
  if (acc==12345) base[0]=acc;
}
__global__ void k_copy(const uint4* a, uint4* b, size_t n){
  for (size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  uint32_t* out; CK(cudaMalloc(&out, 1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // smem
  for (int entries : {4096, 16384, 49152/1*1}) {
    int mask = 1; while (mask < entries) mask <<= 1; mask -= 1; if (mask+1 > 32768) mask = 32767;
    size_t smem = (size_t)(mask+1)*4; if (smem < 8192) smem = 8192;
    for (int tpb : {256, 512, 1024}) {
      int ctas_per_sm = 1;
      CK(cudaFuncSetAttribute(k_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024));
      CK(cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024));
      CK(cudaFuncSetAttribute(k_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024));
      CK(cudaFuncSetAttribute(k_smem<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024));
      int iters = 4096;
      int grid = sms*ctas_per_sm*2;
      const char* names[4]={"smem_red_u32","smem_atom_ret_u32","smem_red_u64","smem_lds_u32"};
      for (int mode=0; mode<4; mode++){
        for (int rep=0; rep<2; rep++){
          cudaEventRecord(e0);
          if(mode==0) k_smem<0><<<grid,tpb,smem>>>(out,iters,mask);
          if(mode==1) k_smem<1><<<grid,tpb,smem>>>(out,iters,mask);
          if(mode==2) k_smem<2><<<grid,tpb,smem>>>(out,iters,mask);
          if(mode==3) k_smem<3><<<grid,tpb,smem>>>(out,iters,mask);
          cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
          cudaEventElapsedTime(&ms,e0,e1);
        }
        double ops = (double)grid*tpb*iters;
        printf("%-18s entries=%6d tpb=%4d : %8.1f Gop/s  (%.3f ms)\n", names[mode], mask+1, tpb, ops/ms/1e6, ms);
      }
    }
  }
  // global atomics
  size_t big = (size_t)1<<30; uint32_t* g; CK(cudaMalloc(&g, big*4)); CK(cudaMemset(g,0,big*4));
  struct Cfg{ size_t per_cta_entries; int shared; const char* name; };
  Cfg cfgs[] = {{1<<14,0,"per-CTA 64KB rows"},{1<<18,0,"per-CTA 1MB rows"},{1<<20,0,"per-CTA 4MB rows"},{1<<20,1,"one 4MB row"},{1<<24,1,"one 64MB row"},{(size_t)1<<30,1,"one 4GB row"}};
  for (auto c : cfgs){
    int grid = sms*4, tpb=256, iters=1024;
    if (!c.shared && (size_t)grid*c.per_cta_entries > big) grid = big / c.per_cta_entries;
    const char* names[3]={"glob_red_u32","glob_atom_ret_u32","glob_red_u64"};
    for (int mode=0; mode<3; mode++){
      for (int rep=0; rep<2; rep++){
        cudaEventRecord(e0);
        if(mode==0) k_glob<0><<<grid,tpb>>>(g,c.per_cta_entries-1,c.shared,iters);
        if(mode==1) k_glob<1><<<grid,tpb>>>(g,c.per_cta_entries-1,c.shared,iters);
        if(mode==2) k_glob<2><<<grid,tpb>>>(g,c.per_cta_entries-1,c.shared,iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms,e0,e1);
      }
      double ops = (double)grid*tpb*iters;
      printf("%-18s %-20s grid=%d : %8.1f Gop/s (%.3f ms)\n", names[mode], c.name, grid, ops/ms/1e6, ms);
    }
  }
  // copy bandwidth
  size_t nbytes = (size_t)2<<30; uint4 *a,*b; CK(cudaMalloc(&a,nbytes)); CK(cudaMalloc(&b,nbytes));
  for (int rep=0;rep<3;rep++){ cudaEventRecord(e0); k_copy<<<sms*8,512>>>(a,b,nbytes/16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);} 
  printf("copy 2GB: %.1f GB/s (r+w)\n", 2.0*nbytes/ms/1e6);
  return 0;
}
