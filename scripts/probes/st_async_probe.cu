// Probe: DSMEM st.async + per-pass mbarrier complete_tx in a 16-CTA cluster.
// Each CTA, for P passes, sends its (rank*1000 + pass) to slot [pass*16 + rank]
// of every CTA's buffer; receivers wait on that pass's barrier (16 x 8 bytes).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void mb_init(uint64_t* bar, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* bar, unsigned b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(b) : "memory");
}
__device__ __forceinline__ bool mb_try(uint64_t* bar, unsigned par) {
  unsigned ok;
  asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
               : "=r"(ok) : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) {
  unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}

template <int VARIANT>
__global__ void __cluster_dims__(16, 1, 1) k_probe(int P, double* out, int* status) {
  cg::cluster_group cl = cg::this_cluster();
  const int r = cl.block_rank();
  __shared__ double buf[64 * 16];
  __shared__ uint64_t bar[64];
  if (threadIdx.x == 0) {
    for (int k = 0; k < P; ++k) mb_init(bar + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < P; ++k) mb_expect(bar + k, 16 * 8);
  }
  __syncthreads();
  cl.sync();
  const unsigned bs = (unsigned)__cvta_generic_to_shared(buf), ms = (unsigned)__cvta_generic_to_shared(bar);
  for (int k = 0; k < P; ++k) {
    if (VARIANT == 2) { if (k > 0) cl.sync(); } else if (k > 0) {
      long spins = 0;
      while (!mb_try(bar + k - 1, 0)) if (++spins > (1L << 24)) { atomicExch(status, 100 + k); return; }
    }
    if (threadIdx.x < 16) {
      const unsigned t = threadIdx.x;
      const double v = r * 1000.0 + k;
      const unsigned wa = mapa(bs, t) + 8u * (unsigned)(k * 16 + r);
      const unsigned ba = mapa(ms, t) + 8u * (unsigned)k;
      if (VARIANT == 2) {
        *cl.map_shared_rank(buf + k * 16 + r, t) = v;
      } else if (VARIANT == 0)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(wa), "d"(v), "r"(ba) : "memory");
      else
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(wa), "l"(__double_as_longlong(v)), "r"(ba) : "memory");
    }
  }
  if (VARIANT == 2) { cl.sync(); } else {
  long spins = 0;
  while (!mb_try(bar + P - 1, 0)) if (++spins > (1L << 24)) { atomicExch(status, 1000 + r); return; }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P * 16; i += blockDim.x) out[r * P * 16 + i] = buf[i];
}

int main() {
  const int P = 34;
  double* out; int* st;
  cudaMalloc(&out, sizeof(double) * 16 * P * 16);
  cudaMalloc(&st, sizeof(int));
  cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int var = 0; var < 3; ++var) {
    cudaMemset(st, 0, sizeof(int));
    cudaMemset(out, 0, sizeof(double) * 16 * P * 16);
    if (var == 0) k_probe<0><<<16, 128>>>(P, out, st); else if (var == 1) k_probe<1><<<16, 128>>>(P, out, st); else k_probe<2><<<16, 128>>>(P, out, st);
    cudaError_t el = cudaGetLastError();
    cudaError_t e = cudaDeviceSynchronize();
    printf("launch: %s\n", cudaGetErrorString(el));
    int hs = 0; cudaMemcpy(&hs, st, sizeof(int), cudaMemcpyDeviceToHost);
    static double h[16 * 34 * 16];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int c = 0; c < 16; ++c) for (int k = 0; k < P; ++k) for (int s = 0; s < 16; ++s)
      if (h[(c * P + k) * 16 + s] != s * 1000.0 + k) ++bad;
    // timing
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int it = 0; it < 100; ++it) { if (var == 0) k_probe<0><<<16, 128>>>(P, out, st); else if (var == 1) k_probe<1><<<16, 128>>>(P, out, st); else k_probe<2><<<16, 128>>>(P, out, st); }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    printf("  sample c0: %g %g %g %g | c5 k3: %g %g\n", h[0], h[1], h[16], h[17], h[(5 * P + 3) * 16 + 2], h[(5 * P + 3) * 16 + 9]);
    printf("variant %d: err=%s status=%d bad=%d  %.2f us per launch (%d passes)\n", var, cudaGetErrorString(e), hs, bad, ms * 10.0f, P);
  }
  return 0;
}
