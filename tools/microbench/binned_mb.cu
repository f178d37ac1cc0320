// Microbenchmark (design exploration, not product): can a row-binned,
// column-sorted layout beat the L1 wavefront bound of CSR x gathers on a
// uniform-random 4M x 4M, 64M nnz fp32 matrix?
//   csr    : 4 lanes per row, register accumulation, random x gathers
//   binned : bins of R rows; entries of a bin sorted by column; packed word =
//            (col_rel << rbits) | row_local; chunks of 2^(32-rbits) columns;
//            accumulation into a shared-memory y segment by MODE:
//            0 = float atomicAdd (CAS loop), 1 = int ATOMS.ADD (proxy), 2 = none
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o binned_mb binned_mb.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("%s: %s\n",#x,cudaGetErrorString(e)); exit(1);}}while(0)

__global__ void csr_kernel(int rows, const int64_t* ro, const int* ci, const float* v, const float* x, float* y){
  int64_t gid = blockIdx.x*(int64_t)blockDim.x + threadIdx.x; int row = gid/4; int lg = threadIdx.x&3;
  float acc=0; if(row<rows){ int64_t b=ro[row], e=ro[row+1];
    for(int64_t k=b+lg;k<e;k+=16){ int c[4]; float a[4]; bool ok[4];
      #pragma unroll
      for(int j=0;j<4;j++){ ok[j]=k+4*j<e; c[j]=ok[j]?__ldg(ci+k+4*j):0; a[j]=ok[j]?__ldg(v+k+4*j):0.f;}
      float xv[4];
      #pragma unroll
      for(int j=0;j<4;j++) xv[j]=ok[j]?__ldg(x+c[j]):0.f;
      #pragma unroll
      for(int j=0;j<4;j++) acc=fmaf(a[j],xv[j],acc);} }
  acc+=__shfl_xor_sync(0xffffffff,acc,1,4); acc+=__shfl_xor_sync(0xffffffff,acc,2,4);
  if(row<rows && lg==0) y[row]=acc;
}

template<int MODE, int NT, int U>
__global__ void __launch_bounds__(NT) binned_kernel(int R, int rbits, int nchunks, const int64_t* choff,
    const uint32_t* pk, const float* v, const float* x, float* y, int rows){
  extern __shared__ float ys[];
  const int b = blockIdx.x;
  for(int i=threadIdx.x;i<R;i+=NT) ys[i]=0.f;
  __syncthreads();
  const int cw = 32 - rbits; const uint32_t rmask = (1u<<rbits)-1;
  const int64_t* co = choff + (int64_t)b*(nchunks+1);
  for(int c=0;c<nchunks;c++){
    const int64_t e0=co[c], e1=co[c+1];
    const float* xc = x + ((int64_t)c<<cw);
    for(int64_t base=e0; base<e1; base += NT*U){
      uint32_t p[U]; float a[U]; float xv[U];
      #pragma unroll
      for(int j=0;j<U;j++){ int64_t e=base+j*NT+threadIdx.x; bool ok=e<e1; p[j]=ok?__ldcs(pk+e):0xffffffffu; a[j]=ok?__ldcs(v+e):0.f; }
      #pragma unroll
      for(int j=0;j<U;j++){ xv[j] = p[j]!=0xffffffffu ? __ldg(xc + (p[j]>>rbits)) : 0.f; }
      #pragma unroll
      for(int j=0;j<U;j++){ if(p[j]!=0xffffffffu){ float pr=a[j]*xv[j]; int rl=p[j]&rmask;
          if(MODE==0) atomicAdd(&ys[rl], pr);
          else if(MODE==1) atomicAdd(reinterpret_cast<int*>(&ys[rl]), __float_as_int(pr));
          else ys[rl&31*0] += 0.f*pr + (pr>1e30f?1.f:0.f); } }
    }
  }
  __syncthreads();
  const int r0 = b*R;
  for(int i=threadIdx.x;i<R && r0+i<rows;i+=NT) y[r0+i]=ys[i];
}


// tile = (row bin b) x (chunk range [c0,c1)); y zeroed beforehand; flush with red.global.add.v4
template<int NT, int U, bool PF>
__global__ void __launch_bounds__(NT,1) tile_kernel(int R, int rbits, int nchunks, int S, const int64_t* choff,
    const uint32_t* pk, const float* v, const float* x, float* y, int rows){
  extern __shared__ float ys[];
  const int b = blockIdx.x / S, s = blockIdx.x % S;
  for(int i=threadIdx.x;i<R;i+=NT) ys[i]=0.f;
  __syncthreads();
  const int cw = 32 - rbits; const uint32_t rmask = (1u<<rbits)-1;
  const int64_t* co = choff + (int64_t)b*(nchunks+1);
  const int c0 = (int)((int64_t)nchunks*s/S), c1=(int)((int64_t)nchunks*(s+1)/S);
  const int64_t e0=co[c0], e1=co[c1];
  // chunk tracked per element: chunk of entry e found by walking (entries sorted by chunk)
  int c = c0; // current chunk for this thread's next element (monotone)
  uint32_t p[U]; float a[U];
  int64_t base=e0;
  auto load=[&](int64_t bs){
    #pragma unroll
    for(int j=0;j<U;j++){ int64_t e=bs+j*NT+threadIdx.x; bool ok=e<e1; p[j]=ok?__ldcs(pk+e):0xffffffffu; a[j]=ok?__ldcs(v+e):0.f; } };
  load(base);
  for(; base<e1; base += NT*U){
    uint32_t q[U]; float aa[U]; int cc[U];
    #pragma unroll
    for(int j=0;j<U;j++){ q[j]=p[j]; aa[j]=a[j]; int64_t e=base+j*NT+threadIdx.x; while(c+1<c1 && co[c+1]<=e) c++; cc[j]=c; }
    if(PF) load(base+NT*U);
    float xv[U];
    #pragma unroll
    for(int j=0;j<U;j++){ xv[j] = q[j]!=0xffffffffu ? __ldg(x + ((int64_t)cc[j]<<cw) + (q[j]>>rbits)) : 0.f; }
    #pragma unroll
    for(int j=0;j<U;j++){ if(q[j]!=0xffffffffu) atomicAdd(&ys[q[j]&rmask], aa[j]*xv[j]); }
    if(!PF) load(base+NT*U);
  }
  __syncthreads();
  const int r0 = b*R;
  for(int i=4*threadIdx.x;i<R;i+=4*NT){ if(r0+i+3<rows){
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(y+r0+i), "f"(ys[i]),"f"(ys[i+1]),"f"(ys[i+2]),"f"(ys[i+3]) : "memory"); } }
}


// v3: entries padded to 32-groups per chunk, optional bank-distinct grouping,
// per-group chunk id (u16); tile = bin (S=1)
template<int NT, int U>
__global__ void __launch_bounds__(NT,1) grp_kernel(int R, int rbits, const int64_t* binoff /*group offsets per bin*/,
    const unsigned short* gchunk, const uint32_t* pk, const float* v, const float* x, float* y, int rows){
  extern __shared__ float ys[];
  const int b = blockIdx.x;
  for(int i=threadIdx.x;i<R;i+=NT) ys[i]=0.f;
  __syncthreads();
  const int cw = 32 - rbits; const uint32_t rmask = (1u<<rbits)-1;
  const int64_t g0=binoff[b], g1=binoff[b+1];
  const int lane=threadIdx.x&31, warp=threadIdx.x>>5; constexpr int NW=NT/32;
  for(int64_t gb=g0+warp; gb<g1; gb += NW*U){
    uint32_t q[U]; float aa[U]; int cc[U];
    #pragma unroll
    for(int j=0;j<U;j++){ int64_t g=gb+j*NW; bool ok=g<g1; int64_t e=g*32+lane;
      q[j]=ok?__ldcs(pk+e):0xffffffffu; aa[j]=ok?__ldcs(v+e):0.f; cc[j]=ok?gchunk[g]:0; }
    float xv[U];
    #pragma unroll
    for(int j=0;j<U;j++){ xv[j] = q[j]!=0xffffffffu ? __ldg(x + ((int64_t)cc[j]<<cw) + (q[j]>>rbits)) : 0.f; }
    #pragma unroll
    for(int j=0;j<U;j++){ if(q[j]!=0xffffffffu) atomicAdd(&ys[q[j]&rmask], aa[j]*xv[j]); }
  }
  __syncthreads();
  const int r0 = b*R;
  for(int i=4*threadIdx.x;i<R;i+=4*NT){ if(r0+i+3<rows){
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(y+r0+i), "f"(ys[i]),"f"(ys[i+1]),"f"(ys[i+2]),"f"(ys[i+3]) : "memory"); } }
}

int main(){
  const int n = 1<<22, rows = 1<<22; const int64_t nnz_t = (int64_t)1<<26;
  std::mt19937_64 g(1); std::uniform_int_distribution<int> uc(0,n-1); std::uniform_real_distribution<float> uv(-1,1);
  // CSR: rows with Poisson-ish degree: assign nnz_t entries to random rows
  std::vector<int64_t> ro(rows+1,0); std::vector<int> rowof(nnz_t);
  for(int64_t k=0;k<nnz_t;k++){ rowof[k]=uc(g); ro[rowof[k]+1]++; }
  for(int i=0;i<rows;i++) ro[i+1]+=ro[i];
  std::vector<int> ci(nnz_t); std::vector<float> vals(nnz_t);
  { std::vector<int64_t> pos(ro.begin(),ro.end()-1); for(int64_t k=0;k<nnz_t;k++){ int64_t p=pos[rowof[k]]++; ci[p]=uc(g); vals[p]=uv(g);} }
  for(int i=0;i<rows;i++) std::sort(ci.begin()+ro[i], ci.begin()+ro[i+1]);
  std::vector<int> rk(nnz_t); for(int i=0;i<rows;i++) for(int64_t k=ro[i];k<ro[i+1];k++) rk[k]=i;
  std::vector<float> xh(n); for(auto& t:xh) t=uv(g);
  int64_t *d_ro; int* d_ci; float *d_v,*d_x,*d_y,*d_flush;
  CK(cudaMalloc(&d_ro,8*(rows+1))); CK(cudaMalloc(&d_ci,4*nnz_t)); CK(cudaMalloc(&d_v,4*nnz_t));
  CK(cudaMalloc(&d_x,4*n)); CK(cudaMalloc(&d_y,4*rows)); CK(cudaMalloc(&d_flush,256<<20));
  CK(cudaMemcpy(d_ro,ro.data(),8*(rows+1),cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_ci,ci.data(),4*nnz_t,cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_v,vals.data(),4*nnz_t,cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_x,xh.data(),4*n,cudaMemcpyHostToDevice));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit=[&](auto f){ float best=1e9, tot=0; for(int it=0;it<8;it++){ cudaMemset(d_flush,it,256<<20); cudaEventRecord(e0); f(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(it>=2){best=std::min(best,ms); tot+=ms;} } return tot/6*1000; };
  float tcsr = timeit([&]{ csr_kernel<<<(rows*4+255)/256,256>>>(rows,d_ro,d_ci,d_v,d_x,d_y); });
  CK(cudaGetLastError());
  std::vector<float> yref(rows); CK(cudaMemcpy(yref.data(),d_y,4*rows,cudaMemcpyDeviceToHost));
  printf("csr 4-lane: %.1f us\n", tcsr);

  for(int R : {16384, 20480, 28672}) for(int bank : {0,1}){
    int rbits=0; while((1<<rbits)<R) rbits++;
    int cw=32-rbits; int nchunks=(n + (1<<cw)-1)>>cw; int B=(rows+R-1)/R;
    std::vector<uint32_t> pk; std::vector<float> bv; std::vector<unsigned short> gch; std::vector<int64_t> binoff(B+1,0);
    pk.reserve(nnz_t*1.05); bv.reserve(nnz_t*1.05);
    for(int b=0;b<B;b++){
      int r0=b*R, r1=std::min(rows,r0+R);
      std::vector<std::pair<int,int64_t>> es; es.reserve(ro[r1]-ro[r0]);
      for(int64_t k=ro[r0];k<ro[r1];k++) es.push_back({ci[k],k});
      std::sort(es.begin(),es.end());
      size_t i=0;
      for(int c=0;c<nchunks;c++){
        size_t j=i; while(j<es.size() && (es[j].first>>cw)==c) j++;
        for(size_t w0=i; w0<j; w0+=256){
          size_t w1=std::min(j,w0+256); size_t cnt=w1-w0; size_t ng=(cnt+31)/32;
          std::vector<int64_t> order;
          if(bank){ std::vector<std::vector<size_t>> bk(32); for(size_t t=w0;t<w1;t++){ int row=rk[es[t].second]-r0; bk[row&31].push_back(t);} 
            std::vector<int64_t> slots(ng*32,-1); std::vector<size_t> left;
            for(size_t g=0;g<ng;g++) for(int q=0;q<32;q++) if(!bk[q].empty()){ slots[g*32+q]=bk[q].back(); bk[q].pop_back(); }
            for(int q=0;q<32;q++) for(auto t:bk[q]) left.push_back(t);
            size_t li=0; for(auto& sl:slots) if(sl<0 && li<left.size()) sl=left[li++];
            order.assign(slots.begin(),slots.end());
          } else { for(size_t t=w0;t<w1;t++) order.push_back(t); while(order.size()%32) order.push_back(-1); }
          for(size_t g=0; g<order.size()/32; g++){ gch.push_back(c);
            for(int q=0;q<32;q++){ int64_t t=order[g*32+q]; if(t<0){ pk.push_back(0xffffffffu); bv.push_back(0);} else {
              int col=es[t].first; int64_t k=es[t].second; int row=rk[k];
              pk.push_back(((uint32_t)(col&((1<<cw)-1))<<rbits)|(uint32_t)(row-r0)); bv.push_back(vals[k]); } } }
        }
        i=j;
      }
      binoff[b+1]=gch.size();
    }
    int64_t ne=pk.size();
    int64_t* d_bo; unsigned short* d_gc; uint32_t* d_pk; float* d_bv;
    CK(cudaMalloc(&d_bo,8*(B+1))); CK(cudaMalloc(&d_gc,2*gch.size())); CK(cudaMalloc(&d_pk,4*ne)); CK(cudaMalloc(&d_bv,4*ne));
    CK(cudaMemcpy(d_bo,binoff.data(),8*(B+1),cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_gc,gch.data(),2*gch.size(),cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_pk,pk.data(),4*ne,cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_bv,bv.data(),4*ne,cudaMemcpyHostToDevice));
    size_t sm=4*(size_t)R;
    auto kt=[&](auto kern, int NT){ CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        return timeit([&]{ cudaMemsetAsync(d_y,0,4*rows); kern<<<B,NT,sm>>>(R,rbits,d_bo,d_gc,d_pk,d_bv,d_x,d_y,rows); }); };
    float a1=kt(grp_kernel<1024,4>,1024);
    std::vector<float> yb2(rows); CK(cudaMemcpy(yb2.data(),d_y,4*rows,cudaMemcpyDeviceToHost));
    double md=0; for(int i=0;i<rows;i++) md=std::max(md,(double)fabsf(yb2[i]-yref[i]));
    float a2=kt(grp_kernel<1024,8>,1024);
    float a3=kt(grp_kernel<512,8>,512);
    float a4=kt(grp_kernel<1024,2>,1024);
    CK(cudaGetLastError());
    printf("grp R=%d bank=%d bins=%d pad=%.3f: NT1024U4 %.1f (maxdiff %.2e) NT1024U8 %.1f NT512U8 %.1f NT1024U2 %.1f\n",R,bank,B,(double)ne/nnz_t,a1,md,a2,a3,a4);
    cudaFree(d_bo); cudaFree(d_gc); cudaFree(d_pk); cudaFree(d_bv);
  }
  return 0;
  for(int R : {28672}){
    int rbits=0; while((1<<rbits)<R) rbits++;
    int cw=32-rbits; int nchunks=(n + (1<<cw)-1)>>cw; int B=(rows+R-1)/R;
    // build binned layout on host
    std::vector<std::vector<uint64_t>> bins(B); // key = col<<32 | idx
    std::vector<int64_t> choff((int64_t)B*(nchunks+1));
    std::vector<uint32_t> pk(nnz_t); std::vector<float> bv(nnz_t);
    int64_t w=0;
    for(int b=0;b<B;b++){
      std::vector<std::pair<int,int64_t>> es; // (col, k)
      int r0=b*R, r1=std::min(rows,r0+R);
      es.reserve(ro[r1]-ro[r0]);
      for(int64_t k=ro[r0];k<ro[r1];k++) es.push_back({ci[k],k});
      std::sort(es.begin(),es.end());
      int64_t* co=&choff[(int64_t)b*(nchunks+1)];
      int c=0; co[0]=w;
      // need row of k: search
      for(auto& pr:es){ int col=pr.first; while((col>>cw)>c){ c++; co[c]=w; }
        int64_t k=pr.second; int row = rk[k];
        pk[w]=((uint32_t)(col & ((1<<cw)-1))<<rbits) | (uint32_t)(row-r0); bv[w]=vals[k]; w++; }
      while(c<nchunks){ c++; co[c]=w; }
    }
    int64_t* d_co; uint32_t* d_pk; float* d_bv;
    CK(cudaMalloc(&d_co,8*choff.size())); CK(cudaMalloc(&d_pk,4*nnz_t)); CK(cudaMalloc(&d_bv,4*nnz_t));
    CK(cudaMemcpy(d_co,choff.data(),8*choff.size(),cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_pk,pk.data(),4*nnz_t,cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_bv,bv.data(),4*nnz_t,cudaMemcpyHostToDevice));
    size_t sm = 4*(size_t)R;
    auto run=[&](auto kern, int NT){ CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      return timeit([&]{ kern<<<B,NT,sm>>>(R,rbits,nchunks,d_co,d_pk,d_bv,d_x,d_y,rows); }); };
    float t0=run(binned_kernel<0,512,4>,512);
    std::vector<float> yb(rows); CK(cudaMemcpy(yb.data(),d_y,4*rows,cudaMemcpyDeviceToHost));
    double maxd=0; for(int i=0;i<rows;i++) maxd=std::max(maxd,(double)fabsf(yb[i]-yref[i]));
    float t0b=run(binned_kernel<0,1024,4>,1024);
    float t1=run(binned_kernel<1,512,4>,512);
    float t2=run(binned_kernel<2,512,4>,512);
    float t2b=run(binned_kernel<2,512,8>,512);
    for(int S : {1,2,4}){
      auto kt=[&](auto kern, int NT){ CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        return timeit([&]{ cudaMemsetAsync(d_y,0,4*rows); kern<<<B*S,NT,sm>>>(R,rbits,nchunks,S,d_co,d_pk,d_bv,d_x,d_y,rows); }); };
      float a1=kt(tile_kernel<1024,4,true>,1024);
      std::vector<float> yb2(rows); CK(cudaMemcpy(yb2.data(),d_y,4*rows,cudaMemcpyDeviceToHost));
      double md=0; for(int i=0;i<rows;i++) md=std::max(md,(double)fabsf(yb2[i]-yref[i]));
      float a2=kt(tile_kernel<1024,8,true>,1024);
      float a3=kt(tile_kernel<512,8,true>,512);
      float a4=kt(tile_kernel<1024,4,false>,1024);
      printf("  tile R=%d S=%d grid=%d: NT1024U4pf %.1f (maxdiff %.2e) NT1024U8pf %.1f NT512U8pf %.1f NT1024U4 %.1f\n",R,S,B*S,a1,md,a2,a3,a4);
    }
    CK(cudaGetLastError());
    printf("R=%d bins=%d chunks=%d: fatomic512 %.1f us (maxdiff %.2e) fatomic1024 %.1f | intatomic %.1f | noacc U4 %.1f U8 %.1f\n",R,B,nchunks,t0,maxd,t0b,t1,t2,t2b);
    cudaFree(d_co); cudaFree(d_pk); cudaFree(d_bv);
  }
  return 0;
}
