// exp_nonpos_test.cu — accuracy of topk.cu's exp_nonpos (copied here verbatim) against the host exp.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/exp_nonpos_test tools/exp_nonpos_test.cu
#include <cstdio>
#include <cmath>
#include <random>
#include <vector>
__constant__ double c_exp2_64[64];  // 2^(i/64), from the host's exp2

// e^a for a ≤ 0: a = (64k + i)·ln2/64 + r, |r| ≤ ln2/128; e^r by its
// degree-5 Taylor polynomial (truncation ≤ 4e-17), times 2^(i/64) from the
// table, times 2^k by exponent arithmetic.  11 FP64 operations against ~18
// in libdevice's exp; ≤ 2 ulp.  a < −707 → 0 (keeps the result normal:
// such entries are < 1e-307 of the diagonal).
__device__ __forceinline__ double exp_nonpos(double a, const double* tab) {
  constexpr double kInvLn2x64 = 92.33248261689366;            // 64/ln2
  constexpr double kLn2by64Hi = 0.010830424695086549;         // ln2/64, 33 bits (n·hi exact)
  constexpr double kLn2by64Lo = 1.162596423439437e-12;        // ln2/64 − hi
  constexpr double kShift = 6755399441055744.0;               // 1.5·2^52
  if (a < -707.0) return 0.0;
  const double kd = fma(a, kInvLn2x64, kShift);
  const int n = __double2loint(kd);                           // round(a·64/ln2)
  const double kf = kd - kShift;
  double r = fma(kf, -kLn2by64Hi, a);
  r = fma(kf, -kLn2by64Lo, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double v = p * tab[n & 63];
  // v ∈ [0.99, 2): add n >> 6 (≤ 0, ≥ −1020) to the exponent
  return __hiloint2double(__double2hiint(v) + ((n >> 6) << 20), __double2loint(v));
}
__global__ void k(const double* a, double* o, int n){ __shared__ double tab[64]; if(threadIdx.x<64) tab[threadIdx.x]=c_exp2_64[threadIdx.x]; __syncthreads(); int i=blockIdx.x*blockDim.x+threadIdx.x; if(i<n) o[i]=exp_nonpos(a[i],tab);}
int main(){ int n=1<<20; double tab[64]; for(int i=0;i<64;++i) tab[i]=std::exp2(i/64.0); cudaMemcpyToSymbol(c_exp2_64,tab,sizeof tab);
 std::vector<double> a(n),o(n); std::mt19937_64 g(1); std::uniform_real_distribution<double> u(-750,0); for(int i=0;i<n;++i) a[i]= i<n/2? u(g) : -std::ldexp(1.0, -(i%60)) * (1+u(g)/-750);
 double *da,*dout; cudaMalloc(&da,n*8); cudaMalloc(&dout,n*8); cudaMemcpy(da,a.data(),n*8,cudaMemcpyHostToDevice); k<<<n/256,256>>>(da,dout,n); cudaMemcpy(o.data(),dout,n*8,cudaMemcpyDeviceToHost);
 double worst=0; for(int i=0;i<n;++i){ double r=std::exp(a[i]); if(a[i]<-707) { if(o[i]!=0) {printf("nz %g\n",a[i]);} continue;} double e=std::fabs(o[i]-r)/r; if(e>worst) worst=e;} printf("worst rel %.3e (%.2f ulp)\n",worst,worst/1.11e-16); }
