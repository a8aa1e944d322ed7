// K7 — FGMRES(m) vector kernels (sm_100a, fp64): P:L354, P:L433-435 (flexible GMRES, right preconditioned),
// modified Gram–Schmidt with the update of step i-1 fused into the dot of step i, deterministic two-level
// reductions (fixed grid, fixed-order last-block combine), Givens rotations and back substitution on device
// (readings A2-A4, A35).
#include "stgmg_internal.cuh"

namespace stgmg {

constexpr int RED_BLOCKS = 1184;   // 8 x 148 SMs
constexpr int RED_THREADS = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  __syncthreads();
  return s;   // valid in thread 0
}

// w <- w - (*hprev) vprev (if vprev), then out = <w, vnext> (vnext == nullptr: <w, w>; do_sqrt: sqrt), summed over
// the DoFs with mask[i] != 0 (owned DoFs of the x-slab decomposition; mask == nullptr: all).
__global__ void __launch_bounds__(RED_THREADS) mgs_dot_kernel(double* __restrict__ w, const double* __restrict__ vprev,
                                                              const double* __restrict__ hprev,
                                                              const double* __restrict__ vnext, long long n,
                                                              double* __restrict__ partials, unsigned* counter,
                                                              double* __restrict__ out, int do_sqrt,
                                                              const unsigned char* __restrict__ mask) {
  pdl_trigger();
  __shared__ double sh[32];
  __shared__ bool last;
  pdl_wait();
  const double coef = vprev ? *hprev : 0.0;
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double wi = w[i];
    if (vprev) {
      wi = fma(-coef, vprev[i], wi);
      w[i] = wi;
    }
    const double vi = vnext ? vnext[i] : wi;
    if (!mask || mask[i]) s = fma(wi, vi, s);
  }
  const double bsum = block_sum(s, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bsum;
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double p = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) p += ((volatile double*)partials)[i];
    const double tot = block_sum(p, sh);
    if (threadIdx.x == 0) {
      *out = do_sqrt ? sqrt(tot) : tot;
      *counter = 0u;
    }
  }
}

cudaError_t launch_mgs_dot(double* w, const double* vprev, const double* hprev, const double* vnext, long long n,
                           double* partials, unsigned* counter, double* out, int do_sqrt, const unsigned char* mask,
                           cudaStream_t s) {
  return launch_pdl(mgs_dot_kernel, dim3(RED_BLOCKS), dim3(RED_THREADS), 0, s, w, vprev, hprev, vnext, n, partials,
                    counter, out, do_sqrt, mask);
}

__global__ void sqrt_kernel(double* v) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *v = sqrt(*v);
}

cudaError_t launch_sqrt(double* v, cudaStream_t s) {
  sqrt_kernel<<<1, 32, 0, s>>>(v);
  return cudaGetLastError();
}

// y = x * (*sc) (invert: y = x / *sc)
__global__ void scale_kernel(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ sc,
                             int invert, long long n) {
  pdl_trigger();
  pdl_wait();
  const double f = invert ? 1.0 / *sc : *sc;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = x[i] * f;
}

cudaError_t launch_scale(double* y, const double* x, const double* sc, int invert, long long n, cudaStream_t s) {
  return launch_pdl(scale_kernel, dim3(RED_BLOCKS), dim3(RED_THREADS), 0, s, y, x, sc, invert, n);
}

// Givens step for Arnoldi column j of H (column-major, ldh = m+1).  scal[0] = |g_{j+1}|, scal[1] = h_{j+1,j}.
__global__ void givens_kernel(double* H, int ldh, double* cs, double* sn, double* gv, int j, double* scal) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double* h = H + (long long)j * ldh;
  const double hn = h[j + 1];
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * h[i] + sn[i] * h[i + 1];
    h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
    h[i] = t;
  }
  const double rho = hypot(h[j], hn);
  cs[j] = h[j] / rho;
  sn[j] = hn / rho;
  h[j] = rho;
  h[j + 1] = 0.0;
  gv[j + 1] = -sn[j] * gv[j];
  gv[j] = cs[j] * gv[j];
  scal[0] = fabs(gv[j + 1]);
  scal[1] = hn;
}

cudaError_t launch_givens(double* H, int ldh, double* cs, double* sn, double* gv, int j, double* scal, cudaStream_t s) {
  givens_kernel<<<1, 32, 0, s>>>(H, ldh, cs, sn, gv, j, scal);
  return cudaGetLastError();
}

// Device-resident Arnoldi loop (one CUDA graph per restart cycle, one IF node per step j): the Givens step of column
// j also counts the step (ctl[0]: Arnoldi steps of the solve, ctl[1]: steps of this cycle = j + 1) and decides, with
// the host loop's test (|g_{j+1}| <= target, breakdown h_{j+1,j} <= 1e-14 beta_cycle, maxit; scal[4] = target,
// scal[5] = maxit, scal[2] = beta_cycle), whether step j + 1 runs: cudaGraphSetConditional on its IF node's handle.
__global__ void givens_cond_kernel(double* H, int ldh, double* cs, double* sn, double* gv, int j, double* scal, int* ctl,
                                   int has_next, cudaGraphConditionalHandle next) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double* h = H + (long long)j * ldh;
  const double hn = h[j + 1];
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * h[i] + sn[i] * h[i + 1];
    h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
    h[i] = t;
  }
  const double rho = hypot(h[j], hn);
  cs[j] = h[j] / rho;
  sn[j] = hn / rho;
  h[j] = rho;
  h[j + 1] = 0.0;
  gv[j + 1] = -sn[j] * gv[j];
  gv[j] = cs[j] * gv[j];
  scal[0] = fabs(gv[j + 1]);
  scal[1] = hn;
  const int its = ctl[0] + 1;
  ctl[0] = its;
  ctl[1] = j + 1;
  const bool stop = scal[0] <= scal[4] || hn <= 1e-14 * scal[2] || its >= (int)scal[5];
  if (has_next) cudaGraphSetConditional(next, stop ? 0u : 1u);
}
cudaError_t launch_givens_cond(double* H, int ldh, double* cs, double* sn, double* gv, int j, double* scal, int* ctl,
                               int has_next, cudaGraphConditionalHandle next, cudaStream_t s) {
  givens_cond_kernel<<<1, 32, 0, s>>>(H, ldh, cs, sn, gv, j, scal, ctl, has_next, next);
  return cudaGetLastError();
}
// Back substitution and x update with the step count of the cycle read from the device (ctl[1]).
__global__ void backsub_ctl_kernel(const double* H, int ldh, const double* gv, double* y, const int* ctl) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int jn = ctl[1];
  for (int i = jn - 1; i >= 0; --i) {
    double s = gv[i];
    for (int l = i + 1; l < jn; ++l) s -= H[(long long)l * ldh + i] * y[l];
    y[i] = s / H[(long long)i * ldh + i];
  }
}
cudaError_t launch_backsub_ctl(const double* H, int ldh, const double* gv, double* y, const int* ctl, cudaStream_t s) {
  backsub_ctl_kernel<<<1, 32, 0, s>>>(H, ldh, gv, y, ctl);
  return cudaGetLastError();
}
__global__ void update_x_ctl_kernel(double* __restrict__ x, const double* __restrict__ Z, const double* __restrict__ y,
                                    const int* __restrict__ ctl, long long n) {
  pdl_trigger();
  pdl_wait();
  const int jn = ctl[1];
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = x[i];
    for (int j = 0; j < jn; ++j) s = fma(y[j], Z[(long long)j * n + i], s);
    x[i] = s;
  }
}
cudaError_t launch_update_x_ctl(double* x, const double* Z, const double* y, const int* ctl, long long n,
                                cudaStream_t s) {
  return launch_pdl(update_x_ctl_kernel, dim3(RED_BLOCKS), dim3(RED_THREADS), 0, s, x, Z, y, ctl, n);
}

// Back substitution H(0:jn,0:jn) y = g(0:jn).
__global__ void backsub_kernel(const double* H, int ldh, const double* gv, double* y, int jn) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = jn - 1; i >= 0; --i) {
    double s = gv[i];
    for (int l = i + 1; l < jn; ++l) s -= H[(long long)l * ldh + i] * y[l];
    y[i] = s / H[(long long)i * ldh + i];
  }
}

cudaError_t launch_backsub(const double* H, int ldh, const double* gv, double* y, int jn, cudaStream_t s) {
  backsub_kernel<<<1, 32, 0, s>>>(H, ldh, gv, y, jn);
  return cudaGetLastError();
}

// x += sum_j y_j Z_j
__global__ void update_x_kernel(double* __restrict__ x, const double* __restrict__ Z, const double* __restrict__ y,
                                int jn, long long n) {
  pdl_trigger();
  pdl_wait();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = x[i];
    for (int j = 0; j < jn; ++j) s = fma(y[j], Z[(long long)j * n + i], s);
    x[i] = s;
  }
}

cudaError_t launch_update_x(double* x, const double* Z, const double* y, int jn, long long n, cudaStream_t s) {
  return launch_pdl(update_x_kernel, dim3(RED_BLOCKS), dim3(RED_THREADS), 0, s, x, Z, y, jn, n);
}

__global__ void noop_kernel(int n, double* out) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x + blockIdx.x * blockDim.x < n && out) out[threadIdx.x] = 0.0;
}

cudaError_t launch_noop(int blocks, cudaStream_t s) {
  return launch_pdl(noop_kernel, dim3(blocks), dim3(128), 0, s, 0, (double*)nullptr);
}

__global__ void set_scalar_kernel(double* dst, const double* src) {
  if (threadIdx.x == 0) *dst = *src;
}

cudaError_t launch_set_scalar(double* dst, const double* src, cudaStream_t s) {
  set_scalar_kernel<<<1, 32, 0, s>>>(dst, src);
  return cudaGetLastError();
}

__global__ void identity_kernel(double* X, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) X[i * n + i] = 1.0;
}

cudaError_t launch_identity(double* X, long long n, cudaStream_t s) {
  identity_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(X, n);
  return cudaGetLastError();
}

}  // namespace stgmg
