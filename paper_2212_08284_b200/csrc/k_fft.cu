// ANKH-FFT far field (Alg. 4-5, Thm. 1,
// Cor. 1 and 3; SPEC.md `fftengine`) -- the paper's equispaced-grid engine,
// an alternative to the SVD-compressed M2L of the drop-in path (no reference
// code exists for it; oracle/fft_engine.py restates it for the tests):
//
//   v_c = (E x E x E) Q_c          leaf Chebyshev expansions re-interpolated
//                                  onto an equispaced L_u grid (E[k, l] =
//                                  U_k(c_l), fmm.cpp:421-425's transfer)
//   F   = 1/2 v^T A v              A: H(r) = erfc_screen(xi r)/r between the
//                                  equispaced nodes of every leaf pair that is
//                                  not adjacent (|D|_inf >= 2, images
//                                  |I|_inf <= 1) -- two-level block Toeplitz
//       = 1/(2m) sum_k Re(diag_k) |w_k|^2,  w = DFT6(pad(v))   (Cor. 3)
//
// The 6-D transform is separable: per leaf, the three node axes (L_u inputs,
// P_n = 2 L_u - 1 outputs, the last axis half-complex since v is real:
// NF = P_n P_n L_u frequencies) in one CTA; then the three cell axes (n inputs,
// P_c = 2n - 1 outputs) as batched line transforms over a [c1][c2][c3][nf]
// array whose node-frequency index is innermost (every line access is
// coalesced); the last cell axis is fused with the spectral weighting and the
// energy sum (one partial per CTA, summed by k_finalize in fixed order).
// The plan precompute runs the same transforms on the circulant generator
// (k_fft_gen_node + three dense line passes, the last keeping Re).
#include "kernels.cuh"

namespace ankh_b200 {

namespace {

constexpr double kTwoOverSqrtPiF = 1.1283791670955125739;

__device__ __forceinline__ double erfc_screen_f(double z) {
  // kernel.cpp:14-23, 48-51 (as k_periodic.cu)
  if (z >= 0.0 && z <= 0.5) {
    const double z2 = z * z;
    double term = z, sum = 0.0;
#pragma unroll
    for (int n = 0; n < 13; ++n) {
      sum += term / (2 * n + 1);
      term *= -z2 / (n + 1);
    }
    return 1.0 - kTwoOverSqrtPiF * sum;
  }
  return erfc(z);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

// Node-axis transforms of one real Lu^3 (or Pn^3, dense) block held in
// shared memory (x-major: [a][b][c]), into NF = Pn Pn Lu complex values in
// the order nf = (kx Pn + ky) Lu + kz.  nin: input length per axis (Lu for
// leaf values, Pn for the generator); tw[j] = exp(-2 pi i j / Pn).
__device__ void node_dft(const double* __restrict__ v, int nin, int Lu, int Pn, const double2* __restrict__ tw,
                         double2* __restrict__ s1, double2* __restrict__ s2, double2* __restrict__ out) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // z: real -> half complex, [a][b][kz]
  for (int e = tid; e < nin * nin * Lu; e += nt) {
    const int kz = e % Lu, ab = e / Lu;
    const double* x = v + ab * nin;
    double2 acc = make_double2(0.0, 0.0);
    int ph = 0;
    for (int c = 0; c < nin; ++c) {
      const double2 t = tw[ph];
      acc.x = fma(x[c], t.x, acc.x);
      acc.y = fma(x[c], t.y, acc.y);
      ph += kz;
      if (ph >= Pn) ph -= Pn;
    }
    s1[e] = acc;
  }
  __syncthreads();
  // y: [a][ky][kz]
  for (int e = tid; e < nin * Pn * Lu; e += nt) {
    const int kz = e % Lu, ky = (e / Lu) % Pn, a = e / (Lu * Pn);
    double2 acc = make_double2(0.0, 0.0);
    int ph = 0;
    for (int b = 0; b < nin; ++b) {
      cmac(acc, s1[(a * nin + b) * Lu + kz], tw[ph]);
      ph += ky;
      if (ph >= Pn) ph -= Pn;
    }
    s2[e] = acc;
  }
  __syncthreads();
  // x: [kx][ky][kz]
  for (int e = tid; e < Pn * Pn * Lu; e += nt) {
    const int kyz = e % (Pn * Lu), kx = e / (Pn * Lu);
    double2 acc = make_double2(0.0, 0.0);
    int ph = 0;
    for (int a = 0; a < nin; ++a) {
      cmac(acc, s2[a * Pn * Lu + kyz], tw[ph]);
      ph += kx;
      if (ph >= Pn) ph -= Pn;
    }
    out[e] = acc;
  }
}

constexpr int kNodeThreads = 128;

// Evaluation: one CTA per leaf (Morton m).  Q (Lc^3, the P2M row) -> v =
// (E x E x E) Q (Lu^3) -> node DFT -> X[lex cell][nf].
__global__ void __launch_bounds__(kNodeThreads) k_fft_leaf(const double* __restrict__ exp_leaf, int KS, int depth,
                                                           int Lc, int Lu, const double* __restrict__ E,
                                                           double2* __restrict__ X) {
  extern __shared__ __align__(16) double sm[];
  const int Pn = 2 * Lu - 1, NF = Pn * Pn * Lu;
  const int Kc = Lc * Lc * Lc;
  const int big = (max(Kc, max(Lu * Lc * Lc, Lu * Lu * Lc)) + 1) & ~1;  // transfer stages (even: 16-B alignment below)
  double* q = sm;                    // Kc
  double* t1 = q + big;              // Lu Lc Lc  (x transferred)
  double* t2 = t1 + big;             // Lu Lu Lc
  double* v = t2 + big;              // Lu^3
  double2* tw = reinterpret_cast<double2*>(v + ((Lu * Lu * Lu + 1) & ~1));  // Pn
  double2* s1 = tw + ((Pn + 1) & ~1);                                       // Lu Lu Lu
  double2* s2 = s1 + Lu * Lu * Lu;                                          // Lu Pn Lu
  double2* o = s2 + Lu * Pn * Lu;                                           // NF
  const int tid = threadIdx.x;
  const unsigned m = blockIdx.x;
  const int n = 1 << depth;
  const unsigned lex = (morton_compact3(m >> 2) * n + morton_compact3(m >> 1)) * n + morton_compact3(m);
  ANKH_DASSERT(lex < static_cast<unsigned>(n * n * n) && Lu >= 2 && Lc >= 2);
  for (int e = tid; e < Kc; e += kNodeThreads) q[e] = exp_leaf[static_cast<std::size_t>(m) * KS + e];
  for (int j = tid; j < Pn; j += kNodeThreads) {
    double s, c;
    sincospi(-2.0 * j / Pn, &s, &c);
    tw[j] = make_double2(c, s);
  }
  __syncthreads();
  // x: t1[i][b][c] = sum_a E[i][a] q[a][b][c]
  for (int e = tid; e < Lu * Lc * Lc; e += kNodeThreads) {
    const int bc = e % (Lc * Lc), i = e / (Lc * Lc);
    double acc = 0.0;
    for (int a = 0; a < Lc; ++a) acc = fma(E[i * Lc + a], q[a * Lc * Lc + bc], acc);
    t1[e] = acc;
  }
  __syncthreads();
  // y: t2[i][j][c] = sum_b E[j][b] t1[i][b][c]
  for (int e = tid; e < Lu * Lu * Lc; e += kNodeThreads) {
    const int c = e % Lc, j = (e / Lc) % Lu, i = e / (Lc * Lu);
    double acc = 0.0;
    for (int b = 0; b < Lc; ++b) acc = fma(E[j * Lc + b], t1[(i * Lc + b) * Lc + c], acc);
    t2[e] = acc;
  }
  __syncthreads();
  // z: v[i][j][k] = sum_c E[k][c] t2[i][j][c]
  for (int e = tid; e < Lu * Lu * Lu; e += kNodeThreads) {
    const int k = e % Lu, ij = e / Lu;
    double acc = 0.0;
    for (int c = 0; c < Lc; ++c) acc = fma(E[k * Lc + c], t2[ij * Lc + c], acc);
    v[e] = acc;
  }
  __syncthreads();
  node_dft(v, Lu, Lu, Pn, tw, s1, s2, o);
  __syncthreads();
  double2* dst = X + static_cast<std::size_t>(lex) * NF;
  for (int e = tid; e < NF; e += kNodeThreads) dst[e] = o[e];
}

__device__ __forceinline__ double kernel_h(double r, double xi) { return erfc_screen_f(xi * r) / r; }

// Precompute: one CTA per cell offset (cx, cy, cz) of the (Pc)^3 embedding:
// the generator over the Pn^3 node offsets (27 images when periodic, masked
// to the non-adjacent leaf pairs), then its node DFT -> Y[cell][nf].
__global__ void __launch_bounds__(kNodeThreads) k_fft_gen_node(int depth, int Lu, double rb, double xi, int periodic,
                                                               double2* __restrict__ Y) {
  extern __shared__ __align__(16) double sm[];
  const int n = 1 << depth, Pc = 2 * n, Pn = 2 * Lu - 1, NF = Pn * Pn * Lu;
  double* g = sm;                                               // Pn^3
  double2* tw = reinterpret_cast<double2*>(g + ((Pn * Pn * Pn + 1) & ~1));  // Pn
  double2* s1 = tw + ((Pn + 1) & ~1);                           // Pn Pn Lu
  double2* s2 = s1 + Pn * Pn * Lu;                              // Pn Pn Lu
  double2* o = s2 + Pn * Pn * Lu;                               // NF
  const int tid = threadIdx.x;
  const int cell = blockIdx.x;
  const int ix = cell / (Pc * Pc), iy = (cell / Pc) % Pc, iz = cell % Pc;
  // circulant embedding of size Pc = 2n per cell axis: offsets 0..n-1 at
  // their index, -(n-1)..-1 at index + 2n; index n is outside the Toeplitz
  // block (any value embeds it: zero)
  const bool unused = ix == n || iy == n || iz == n;
  const int dcx = ix < n ? ix : ix - Pc, dcy = iy < n ? iy : iy - Pc, dcz = iz < n ? iz : iz - Pc;
  const double rad = rb / n, h = 2.0 * rad / (Lu - 1);
  for (int j = tid; j < Pn; j += kNodeThreads) {
    double s, c;
    sincospi(-2.0 * j / Pn, &s, &c);
    tw[j] = make_double2(c, s);
  }
  const int I0 = periodic ? -1 : 0, I1 = periodic ? 1 : 0;
  for (int e = tid; e < Pn * Pn * Pn; e += kNodeThreads) {
    const int a = e / (Pn * Pn), b = (e / Pn) % Pn, c = e % Pn;
    const int dnx = a < Lu ? a : a - Pn, dny = b < Lu ? b : b - Pn, dnz = c < Lu ? c : c - Pn;
    double acc = 0.0;
    for (int Ix = I0; Ix <= I1; ++Ix)
      for (int Iy = I0; Iy <= I1; ++Iy)
        for (int Iz = I0; Iz <= I1; ++Iz) {
          const int Dx = dcx + n * Ix, Dy = dcy + n * Iy, Dz = dcz + n * Iz;
          if (unused || max(abs(Dx), max(abs(Dy), abs(Dz))) < 2) continue;  // adjacent: the near field's
          const double zx = 2.0 * rad * Dx + h * dnx, zy = 2.0 * rad * Dy + h * dny, zz = 2.0 * rad * Dz + h * dnz;
          acc += kernel_h(sqrt(zx * zx + zy * zy + zz * zz), xi);
        }
    g[e] = acc;
  }
  __syncthreads();
  node_dft(g, Pn, Lu, Pn, tw, s1, s2, o);
  __syncthreads();
  double2* dst = Y + static_cast<std::size_t>(cell) * NF;
  for (int e = tid; e < NF; e += kNodeThreads) dst[e] = o[e];
}

constexpr int kLineLanes = 32, kLineGroups = 8, kLineThreads = kLineLanes * kLineGroups;

// One cell axis of the 3-D transform over an [outer][axis][inner] complex
// array: out[o][k][i] = sum_{j < nin} in[o][j][i] w^(j k), k < P, w = exp(-2 pi
// i / P).  A CTA takes 32 R consecutive inner elements of one outer index and
// all P outputs (lanes = inner: coalesced); a thread keeps R lines x 4 outputs
// in registers, so each staged input and twiddle it loads feeds 4 resp. R
// complex multiply-adds (shared-memory loads would otherwise bound it).
// mode 0 writes complex, mode 1 writes Re (the spectral diagonal), mode 2
// accumulates sum_k mult(nf) D[k][i] |w|^2 into one partial per CTA (nf =
// inner index mod NF; mult = 1 on the kz = 0 half-plane, else 2).
template <int R>
__global__ void __launch_bounds__(kLineThreads) k_fft_line(const double2* __restrict__ in, void* __restrict__ out,
                                                            int nin, int P, long long n_inner, int mode,
                                                            const double* __restrict__ D, int NF, int Lu,
                                                            double* __restrict__ partial, double scale) {
  constexpr int W = kLineLanes * R, S = 4;
  extern __shared__ __align__(16) double2 sx[];  // nin x W, then P twiddles
  double2* tw = sx + nin * W;
  __shared__ double red[kLineThreads];
  const int lane = threadIdx.x & (kLineLanes - 1), grp = threadIdx.x / kLineLanes;
  const long long tiles = (n_inner + W - 1) / W;
  const long long o = blockIdx.x / tiles;
  const long long i0 = (blockIdx.x % tiles) * W + lane;
  for (int j = threadIdx.x; j < P; j += kLineThreads) {
    double s, c;
    sincospi(-2.0 * j / P, &s, &c);
    tw[j] = make_double2(c, s);
  }
  const double2* src = in + o * nin * n_inner;
  for (int j = grp; j < nin; j += kLineGroups)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long i = i0 + kLineLanes * r;
      sx[j * W + lane + kLineLanes * r] = i < n_inner ? src[j * n_inner + i] : make_double2(0.0, 0.0);
    }
  __syncthreads();
  double e = 0.0;
  double mult[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const long long i = i0 + kLineLanes * r;
    mult[r] = (mode == 2 && i < n_inner && (i % NF) % Lu != 0) ? 2.0 : 1.0;
  }
  for (int k0 = grp; k0 < P; k0 += kLineGroups * S) {
    double2 acc[S][R];
    int ph[S], kk[S];
#pragma unroll
    for (int q = 0; q < S; ++q) {
      kk[q] = k0 + kLineGroups * q < P ? k0 + kLineGroups * q : 0;  // past P: computed, discarded
      ph[q] = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) acc[q][r] = make_double2(0.0, 0.0);
    }
    for (int j = 0; j < nin; ++j) {
      double2 x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = sx[j * W + lane + kLineLanes * r];
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const double2 t = tw[ph[q]];
#pragma unroll
        for (int r = 0; r < R; ++r) cmac(acc[q][r], x[r], t);
        ph[q] += kk[q];
        if (ph[q] >= P) ph[q] -= P;
      }
    }
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const int k = k0 + kLineGroups * q;
      if (k >= P) continue;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long i = i0 + kLineLanes * r;
        if (i >= n_inner) continue;
        const long long dst = (o * P + k) * n_inner + i;
        const double2 a = acc[q][r];
        if (mode == 0)
          static_cast<double2*>(out)[dst] = a;
        else if (mode == 1)
          static_cast<double*>(out)[dst] = a.x;
        else
          e = fma(D[dst] * mult[r], fma(a.x, a.x, a.y * a.y), e);
      }
    }
  }
  if (mode != 2) return;
  red[threadIdx.x] = e;
  __syncthreads();
  for (int s = kLineThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = scale * red[0];
}

// Power-of-two line length P (the cell axes, embedding 2n): a radix-2
// decimation-in-frequency FFT of 32 lines per CTA in shared memory
// ([P][32] complex; inputs j >= nin are zero), outputs read back in
// bit-reversed order -- the same three modes as k_fft_line.  HBM-bound: the
// transform costs ~(P/2) log2 P butterflies per line instead of nin P
// multiply-adds.
__global__ void __launch_bounds__(kLineThreads) k_fft_line2(const double2* __restrict__ in, void* __restrict__ out,
                                                             int nin, int P, int logP, long long n_inner, int mode,
                                                             const double* __restrict__ D, int NF, int Lu,
                                                             double* __restrict__ partial, double scale) {
  extern __shared__ __align__(16) double2 sb[];  // P x 32, then P twiddles
  double2* tw = sb + P * kLineLanes;
  __shared__ double red[kLineThreads];
  const int lane = threadIdx.x & (kLineLanes - 1), grp = threadIdx.x / kLineLanes;
  const long long tiles = (n_inner + kLineLanes - 1) / kLineLanes;
  const long long o = blockIdx.x / tiles;
  const long long i = (blockIdx.x % tiles) * kLineLanes + lane;
  const bool ok = i < n_inner;
  ANKH_DASSERT((P & (P - 1)) == 0 && (1 << logP) == P && nin <= P);
  for (int j = threadIdx.x; j < P; j += kLineThreads) {
    double s, c;
    sincospi(-2.0 * j / P, &s, &c);
    tw[j] = make_double2(c, s);
  }
  const double2* src = in + o * nin * n_inner;
  for (int j = grp; j < P; j += kLineGroups)
    sb[j * kLineLanes + lane] = (ok && j < nin) ? src[j * n_inner + i] : make_double2(0.0, 0.0);
  __syncthreads();
  // DIF radix-4 stages on groups of N = P, P/4, ... (span h = N/4; outputs
  // q = 0..3 of each 4-point DFT to sub-block q, twiddled by W_N^(q r) =
  // w^(q r P/N)), then one radix-2 stage when log2 P is odd
  int N = P, logN = logP;
  for (; N >= 4; N >>= 2, logN -= 2) {
    const int h = N >> 2, st = 1 << (logP - logN);  // powers of two: no integer division
    for (int b = grp; b < P / 4; b += kLineGroups) {
      const int r = b & (h - 1), a = ((b - r) << 2) + r;
      double2* x0 = sb + a * kLineLanes + lane;
      const double2 a0 = x0[0], a1 = x0[h * kLineLanes], a2 = x0[2 * h * kLineLanes], a3 = x0[3 * h * kLineLanes];
      const double2 b0 = make_double2(a0.x + a2.x, a0.y + a2.y), b1 = make_double2(a0.x - a2.x, a0.y - a2.y);
      const double2 b2 = make_double2(a1.x + a3.x, a1.y + a3.y);
      const double2 b3 = make_double2(a1.y - a3.y, a3.x - a1.x);  // -i (a1 - a3)
      x0[0] = make_double2(b0.x + b2.x, b0.y + b2.y);
      x0[h * kLineLanes] = cmul(make_double2(b1.x + b3.x, b1.y + b3.y), tw[r * st]);
      x0[2 * h * kLineLanes] = cmul(make_double2(b0.x - b2.x, b0.y - b2.y), tw[2 * r * st]);
      x0[3 * h * kLineLanes] = cmul(make_double2(b1.x - b3.x, b1.y - b3.y), tw[3 * r * st]);
    }
    __syncthreads();
  }
  if (N == 2) {
    for (int b = grp; b < P / 2; b += kLineGroups) {
      double2* x0 = sb + 2 * b * kLineLanes + lane;
      const double2 u = x0[0], v = x0[kLineLanes];
      x0[0] = make_double2(u.x + v.x, u.y + v.y);
      x0[kLineLanes] = make_double2(u.x - v.x, u.y - v.y);
    }
    __syncthreads();
  }
  double e = 0.0;
  const double mult = (mode == 2 && ok && (i % NF) % Lu != 0) ? 2.0 : 1.0;
  for (int k = grp; k < P; k += kLineGroups) {
    if (!ok) continue;
    // storage position of output k: its mixed-radix digits (4, 4, ..., [2]),
    // least significant first, each placing it in a sub-block of its stage
    int rk = 0, rem = k, ls = logP;
    for (; ls >= 2; ls -= 2, rem >>= 2) rk += (rem & 3) << (ls - 2);
    if (ls == 1) rk += rem & 1;
    const double2 a = sb[rk * kLineLanes + lane];
    const long long dst = (o * P + k) * n_inner + i;
    if (mode == 0)
      static_cast<double2*>(out)[dst] = a;
    else if (mode == 1)
      static_cast<double*>(out)[dst] = a.x;
    else
      e = fma(D[dst] * mult, fma(a.x, a.x, a.y * a.y), e);
  }
  if (mode != 2) return;
  red[threadIdx.x] = e;
  __syncthreads();
  for (int s2 = kLineThreads / 2; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2) red[threadIdx.x] += red[threadIdx.x + s2];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = scale * red[0];
}

// lines per thread: the largest R in {4, 2, 1} whose staged block stays
// within ~100 KB (two CTAs per SM)
int line_r(int nin) { return nin <= 48 ? 4 : (nin <= 97 ? 2 : 1); }

std::size_t line_smem(int nin, int P, int R) {
  return sizeof(double2) * (static_cast<std::size_t>(nin) * kLineLanes * R + P);
}

bool pow2(int P) { return P >= 2 && (P & (P - 1)) == 0; }

long long line_blocks(long long n_outer, long long n_inner, int nin, int P) {
  const long long W = pow2(P) ? kLineLanes : kLineLanes * line_r(nin);
  return n_outer * ((n_inner + W - 1) / W);
}

void launch_line(const double2* in, void* out, long long n_outer, int nin, int P, long long n_inner, int mode,
                 const double* D, int NF, int Lu, double* partial, cudaStream_t st, double scale = 1.0) {
  const unsigned grid = static_cast<unsigned>(line_blocks(n_outer, n_inner, nin, P));
  if (pow2(P)) {
    int logP = 0;
    while ((1 << logP) < P) ++logP;
    static std::atomic<unsigned long long> attr2{0};
    smem_opt_in(attr2, k_fft_line2, 200 * 1024);
    k_fft_line2<<<grid, kLineThreads, sizeof(double2) * (static_cast<std::size_t>(P) * kLineLanes + P), st>>>(
        in, out, nin, P, logP, n_inner, mode, D, NF, Lu, partial, scale);
    return;
  }
  const int R = line_r(nin);
  const std::size_t smem = line_smem(nin, P, R);
#define ANKH_LINE(RR)                                                                                   \
  {                                                                                                     \
    static std::atomic<unsigned long long> attr{0};                                                     \
    smem_opt_in(attr, k_fft_line<RR>, 200 * 1024);  /* + 3 KB static: within the 227 KB */           \
    k_fft_line<RR><<<grid, kLineThreads, smem, st>>>(in, out, nin, P, n_inner, mode, D, NF, Lu, partial, \
                                                     scale);                                            \
  }
  if (R == 4)
    ANKH_LINE(4)
  else if (R == 2)
    ANKH_LINE(2)
  else
    ANKH_LINE(1)
#undef ANKH_LINE
}

std::size_t node_smem_leaf(int Lc, int Lu) {
  const int Pn = 2 * Lu - 1, NF = Pn * Pn * Lu, Kc = Lc * Lc * Lc;
  const int big = (std::max(Kc, std::max(Lu * Lc * Lc, Lu * Lu * Lc)) + 1) & ~1;
  return sizeof(double) * (3 * big + ((Lu * Lu * Lu + 1) & ~1)) +
         sizeof(double2) * (((Pn + 1) & ~1) + Lu * Lu * Lu + Lu * Pn * Lu + NF);
}

std::size_t node_smem_gen(int Lu) {
  const int Pn = 2 * Lu - 1, NF = Pn * Pn * Lu;
  return sizeof(double) * ((Pn * Pn * Pn + 1) & ~1) + sizeof(double2) * (((Pn + 1) & ~1) + 2 * Pn * Pn * Lu + NF);
}

}  // namespace

FftShape fft_shape(int depth, int order_equi) {
  FftShape s;
  s.n = 1 << depth;
  s.Pc = 2 * s.n;  // power-of-two circulant embedding (>= 2n - 1): radix-2 cell-axis FFTs
  s.Lu = order_equi;
  s.Pn = 2 * order_equi - 1;
  s.NF = s.Pn * s.Pn * s.Lu;
  s.energy_blocks = line_blocks(1, static_cast<long long>(s.Pc) * s.Pc * s.NF, s.n, s.Pc);
  return s;
}

void launch_fft_precompute(const FftShape& s, int depth, double rb, double xi, int periodic, double2* tmp_a,
                           double2* tmp_b, double* diag, cudaStream_t st) {
  const long long cells = static_cast<long long>(s.Pc) * s.Pc * s.Pc;
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_fft_gen_node, 227 * 1024);  // the device maximum: plans of any order share the attribute
  k_fft_gen_node<<<static_cast<unsigned>(cells), kNodeThreads, node_smem_gen(s.Lu), st>>>(depth, s.Lu, rb, xi,
                                                                                         periodic, tmp_a);
  const long long NF = s.NF, Pc = s.Pc;
  // [cx][cy][cz][nf]: z (outer cx cy, inner nf), y (outer cx, inner cz nf), x (inner cy cz nf) -> Re
  launch_line(tmp_a, tmp_b, Pc * Pc, s.Pc, s.Pc, NF, 0, nullptr, s.NF, s.Lu, nullptr, st);
  launch_line(tmp_b, tmp_a, Pc, s.Pc, s.Pc, Pc * NF, 0, nullptr, s.NF, s.Lu, nullptr, st);
  launch_line(tmp_a, diag, 1, s.Pc, s.Pc, Pc * Pc * NF, 1, nullptr, s.NF, s.Lu, nullptr, st);
}

void launch_fft_far(const FftShape& s, const double* exp_leaf, int KS, int depth, int order_cheb, const double* E,
                    double2* x0, double2* x1, const double* diag, double* partial, cudaStream_t st) {
  // F = 1/(2m) sum_k Re(diag_k) |w_k|^2, m = Pc^3 Pn^3 (the circulant embedding)
  const double m = static_cast<double>(s.Pc) * s.Pc * s.Pc * s.Pn * s.Pn * s.Pn;
  const long long n = s.n, NF = s.NF, Pc = s.Pc;
  const std::size_t smem = node_smem_leaf(order_cheb, s.Lu);
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_fft_leaf, 227 * 1024);
  k_fft_leaf<<<static_cast<unsigned>(n * n * n), kNodeThreads, smem, st>>>(exp_leaf, KS, depth, order_cheb, s.Lu,
                                                                           E, x0);
  // [cx][cy][cz][nf] (cz < n) -> [cx][cy][kz][nf] -> [cx][ky][kz][nf] -> energy over kx
  launch_line(x0, x1, n * n, s.n, s.Pc, NF, 0, nullptr, s.NF, s.Lu, nullptr, st);
  launch_line(x1, x0, n, s.n, s.Pc, Pc * NF, 0, nullptr, s.NF, s.Lu, nullptr, st);
  launch_line(x0, nullptr, 1, s.n, s.Pc, Pc * Pc * NF, 2, diag, s.NF, s.Lu, partial, st, 0.5 / m);
}

}  // namespace ankh_b200
