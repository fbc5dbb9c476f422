// Microbenchmarks for the B200 fp64 particle path.
// Measures: DFMA rate, DMMA rate, DFMA+DMMA concurrency, SHFL.64 rate,
// smem fp64 CAS-atomic rate, REDG.F64 rate, LDS.128 broadcast rate, stream copy.
// Every kernel also records SM cycles (clock64) so results are clock-independent.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

__device__ long long g_cyc[4096];

template<int NCH>
__global__ void k_dfma(double* out, int iters, double a, double b){
  double c[NCH];
  #pragma unroll
  for(int i=0;i<NCH;i++) c[i]=threadIdx.x*1e-3+i;
  long long t0=clock64();
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<NCH;i++) c[i]=fma(c[i],a,b);
  }
  long long t1=clock64();
  double s=0;
  #pragma unroll
  for(int i=0;i<NCH;i++) s+=c[i];
  if(s==1234.5) out[0]=s;
  if(threadIdx.x==0) g_cyc[blockIdx.x]=t1-t0;
}

__global__ void k_dmma(double* out, int iters){
  double a=threadIdx.x*1e-3, b=1.0-threadIdx.x*1e-4;
  double c[8][2];
  #pragma unroll
  for(int i=0;i<8;i++){c[i][0]=0;c[i][1]=0;}
  long long t0=clock64();
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<8;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(c[i][0]),"+d"(c[i][1]) : "d"(a),"d"(b));
  }
  long long t1=clock64();
  double s=0;
  #pragma unroll
  for(int i=0;i<8;i++) s+=c[i][0]+c[i][1];
  if(s==1234.5) out[0]=s;
  if(threadIdx.x==0) g_cyc[blockIdx.x]=t1-t0;
}

// mix: per iteration 8 DMMA + 32 DFMA (per lane)
__global__ void k_mix(double* out, int iters, double x, double y){
  double a=threadIdx.x*1e-3, b=1.0-threadIdx.x*1e-4;
  double c[8][2]; double f[8];
  #pragma unroll
  for(int i=0;i<8;i++){c[i][0]=0;c[i][1]=0;f[i]=i;}
  long long t0=clock64();
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<8;i++){
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(c[i][0]),"+d"(c[i][1]) : "d"(a),"d"(b));
      #pragma unroll
      for(int j=0;j<4;j++) f[i]=fma(f[i],x,y);
    }
  }
  long long t1=clock64();
  double s=0;
  #pragma unroll
  for(int i=0;i<8;i++) s+=c[i][0]+c[i][1]+f[i];
  if(s==1234.5) out[0]=s;
  if(threadIdx.x==0) g_cyc[blockIdx.x]=t1-t0;
}

__global__ void k_shfl(double* out, int iters){
  double v[8];
  #pragma unroll
  for(int i=0;i<8;i++) v[i]=threadIdx.x+i;
  long long t0=clock64();
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<8;i++) v[i]=__shfl_xor_sync(0xffffffffu,v[i],(i+1)&31);
  }
  long long t1=clock64();
  double s=0;
  #pragma unroll
  for(int i=0;i<8;i++) s+=v[i];
  if(s==1234.5) out[0]=s;
  if(threadIdx.x==0) g_cyc[blockIdx.x]=t1-t0;
}

__global__ void k_atoms(double* out, int iters){
  __shared__ double s[4096];
  for(int i=threadIdx.x;i<4096;i+=blockDim.x) s[i]=0;
  __syncthreads();
  long long t0=clock64();
  for(int it=0;it<iters;it++){
    atomicAdd(&s[(threadIdx.x*9+it*33)&4095], 1.0);
  }
  long long t1=clock64();
  __syncthreads();
  if(s[threadIdx.x]==1234.5) out[0]=1;
  if(threadIdx.x==0) g_cyc[blockIdx.x]=t1-t0;
}

__global__ void k_redg(double* out, int iters){
  long long t0=clock64();
  double* base=out+ (size_t)blockIdx.x*8192;
  for(int it=0;it<iters;it++){
    atomicAdd(&base[(threadIdx.x*9+it*33)&8191], 1.0);
  }
  long long t1=clock64();
  if(threadIdx.x==0) g_cyc[blockIdx.x]=t1-t0;
}

__global__ void k_lds(double* out, int iters){
  __shared__ double2 s[512];
  for(int i=threadIdx.x;i<512;i+=blockDim.x) s[i]=make_double2(i,i+1);
  __syncthreads();
  double ax=0, ay=0;
  int idx=(threadIdx.x>>5)&7;  // warp-uniform -> broadcast
  long long t0=clock64();
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int j=0;j<8;j++){ double2 q=s[(idx*8+j+it)&511]; ax+=q.x; ay+=q.y; }
  }
  long long t1=clock64();
  if(ax+ay==1234.5) out[0]=1;
  if(threadIdx.x==0) g_cyc[blockIdx.x]=t1-t0;
}

// stream: read 7 arrays (56 B), write 6 (48 B) per element = particle-update traffic shape
__global__ void k_stream(const double* __restrict__ in, double* __restrict__ o, long n){
  long stride=(long)gridDim.x*blockDim.x;
  for(long i=blockIdx.x*(long)blockDim.x+threadIdx.x;i<n;i+=stride){
    double a0=in[i],a1=in[i+n],a2=in[i+2*n],a3=in[i+3*n],a4=in[i+4*n],a5=in[i+5*n],a6=in[i+6*n];
    o[i]=a0+a6; o[i+n]=a1; o[i+2*n]=a2; o[i+3*n]=a3; o[i+4*n]=a4; o[i+5*n]=a5;
  }
}

static float timeit(void(*launch)(void*), void* arg, int reps){
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(arg); CK(cudaDeviceSynchronize());
  float best=1e30f;
  for(int r=0;r<reps;r++){
    cudaEventRecord(a); launch(arg); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms,a,b); if(ms<best) best=ms;
  }
  return best;
}
static double mean_cyc(int nb){
  static long long h[4096]; cudaMemcpyFromSymbol(h,g_cyc,sizeof(long long)*nb);
  double s=0; for(int i=0;i<nb;i++) s+=h[i]; return s/nb;
}
struct A{double* out; int iters; int nb; int nt;};
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int nsm=p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out,(size_t)nsm*8*8192*sizeof(double)));
  printf("{\"gpu\":\"%s\",\"sms\":%d", p.name, nsm);
  // DFMA: 8 blocks/SM * 256 thr, 16 chains
  { A a{out,4096,nsm*8,256};
    float ms=timeit([](void* v){A* a=(A*)v; k_dfma<16><<<a->nb,a->nt>>>(a->out,a->iters,1.0000001,1e-9);},&a,5);
    double ops=(double)a.nb*a.nt*a.iters*16; double cyc=mean_cyc(a.nb);
    printf(",\"dfma_tflops\":%.2f,\"dfma_per_clk_per_sm\":%.1f,\"dfma_ms\":%.3f,\"dfma_implied_mhz\":%.0f",
      2*ops/ms/1e9, ops/nsm/cyc*1.0, ms, cyc/(ms*1e3)); }
  { A a{out,2048,nsm*8,256};
    float ms=timeit([](void* v){A* a=(A*)v; k_dmma<<<a->nb,a->nt>>>(a->out,a->iters);},&a,5);
    double mmas=(double)a.nb*(a.nt/32)*a.iters*8; double cyc=mean_cyc(a.nb);
    printf(",\"dmma_tflops\":%.2f,\"dmma_warp_instr_per_clk_per_sm\":%.3f",
      mmas*512/ms/1e9, mmas/nsm/cyc); }
  { A a{out,1024,nsm*8,256};
    float ms=timeit([](void* v){A* a=(A*)v; k_mix<<<a->nb,a->nt>>>(a->out,a->iters,1.0000001,1e-9);},&a,5);
    double mmas=(double)a.nb*(a.nt/32)*a.iters*8; double fmas=(double)a.nb*a.nt*a.iters*32;
    printf(",\"mix_ms\":%.3f,\"mix_dmma_tflops\":%.2f,\"mix_dfma_tflops\":%.2f",
      ms, mmas*512/ms/1e9, 2*fmas/ms/1e9); }
  { A a{out,4096,nsm*8,256};
    timeit([](void* v){A* a=(A*)v; k_shfl<<<a->nb,a->nt>>>(a->out,a->iters);},&a,3);
    double sh=(double)(a.nt/32)*8*a.iters*8/ (double)1; double cyc=mean_cyc(a.nb);
    printf(",\"shfl64_warp_instr_per_clk_per_sm\":%.3f", sh/cyc); }
  { A a{out,1024,nsm*4,256};
    timeit([](void* v){A* a=(A*)v; k_atoms<<<a->nb,a->nt>>>(a->out,a->iters);},&a,3);
    double cyc=mean_cyc(a.nb); double ops=(double)a.nt*a.iters*4;
    printf(",\"atoms_f64_lane_ops_per_clk_per_sm\":%.3f", ops/cyc); }
  { A a{out,1024,nsm*4,256};
    float ms=timeit([](void* v){A* a=(A*)v; cudaMemset(a->out,0,(size_t)a->nb*8192*8); k_redg<<<a->nb,a->nt>>>(a->out,a->iters);},&a,3);
    double ops=(double)a.nb*a.nt*a.iters;
    printf(",\"redg_f64_gops_incl_memset\":%.1f", ops/ms/1e6); }
  { A a{out,4096,nsm*8,256};
    timeit([](void* v){A* a=(A*)v; k_lds<<<a->nb,a->nt>>>(a->out,a->iters);},&a,3);
    double cyc=mean_cyc(a.nb); double ops=(double)8*(a.nt/32)*a.iters*8;
    printf(",\"lds128_bcast_warp_instr_per_clk_per_sm\":%.3f", ops/cyc); }
  { long n=1L<<27; double *in,*o; CK(cudaMalloc(&in,n*7*8)); CK(cudaMalloc(&o,n*6*8));
    cudaMemset(in,0,n*7*8);
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float best=1e30f;
    for(int r=0;r<6;r++){ cudaEventRecord(a); k_stream<<<nsm*8,256>>>(in,o,n); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); if(r && ms<best) best=ms;}
    printf(",\"stream_104B_gbs\":%.1f,\"stream_updates_per_s\":%.3e", n*104.0/best/1e6, n/best*1e3);
    cudaFree(in); cudaFree(o); }
  printf("}\n");
  return 0;
}
