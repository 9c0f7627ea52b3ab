// One training step of the encoder-solver network on the device.
//
// The reference ships no trainer; the contract is SPEC.md `[MODULE] trainer`
// (reference SPEC.md:454-507) on the reference's autodiff semantics
// (autodiff.py): MSE of the preconditioner estimate u0 = (h^2/64) net(r)
// against the true error e (paper Eq. 4.10), encoder and solver trained
// jointly, training-mode batch norm (autodiff.py:547-592), the Green spectrum
// rebuilt from the trainable kernel every step with its gradient
// (green.py:55-82), Adam.  The CPU restatement is oracle/train_oracle.py,
// pinned to gradients of the reference autodiff (tests/golden/train.npz).
//
// Data layout: activations NHWC fp32 (channels fastest, coalesced per pixel);
// parameters one flat fp32 vector in netparams.param_spec order (complex
// implicit kernels as (re, im) pairs), with gradient / Adam m / Adam v vectors
// of the same layout.  Every 3x3 convolution, its data gradient and the
// transposed convolution are one gather kernel (k_tr_conv) in either
// correlation or transposed index mode; weight gradients are a pixel-split
// tiled reduction (k_tr_wgrad) with a deterministic partial sum; per-channel
// statistics are two-stage deterministic reductions in double.  The implicit
// layer and the Green-function chain use cuFFT (batched C2C / Z2Z) with own
// kernels for embedding, products and the Wirtinger chain rule.
#include <cufft.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <vector>

#include "../../include/helmsolve_b200.h"
#include "common.cuh"
#include "conv_tc.h"
#include "prof.h"

namespace hs {
namespace {

constexpr double kBnEps = 1e-5;
constexpr double kMomentum = 0.1;  // autodiff.py:555
constexpr double kSpecEps = 1e-5;  // green.py:19

unsigned g1(long long n, int threads = 256) {
  long long g = (n + threads - 1) / threads;
  return (unsigned)(g > 8192 ? 8192 : (g < 1 ? 1 : g));
}

#define GRID_STRIDE(i, n) \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (n); i += (long long)gridDim.x * blockDim.x)

// ------------------------------------------------------------------ 3x3 gather convolution

// out[n, o, co] = sum_{ci, u, v} in[n, pos(o, u, v), ci] * W(co, ci, u, v) (+ bias) (+ addend) (+ out)
//   correlation (trans = 0): pos = s o + (u, v) - 1            -- conv2d forward / tconv data gradient
//   transposed  (trans = 1): pos = (o + 1 - (u, v)) / s if exact -- tconv forward / conv data gradient
// W(co, ci, u, v) = w[co * sco + ci * sci + 3u + v] covers every weight orientation.
struct TrConv {
  const float* x;
  int Hi, Wi, Ci;
  float* y;
  int Ho, Wo, Co;
  const float* w;
  int sco, sci;
  const float* bias;
  const float* addend;
  int trans, s, accumulate, B;
};

constexpr int kConvThreads = 128;
constexpr int kCk = 32;

// PX consecutive output pixels of one row per thread (Wo % PX == 0) x COB output channels:
// weights staged in shared memory per 32-channel slice and read as broadcasts, reused PX times.
template <int COB, int PX>
__global__ void __launch_bounds__(kConvThreads) k_tr_conv(TrConv a) {
  __shared__ __align__(16) float ws[9][kCk][COB];
  const long long npix = (long long)a.B * a.Ho * a.Wo;
  const long long pix = ((long long)blockIdx.x * kConvThreads + threadIdx.x) * PX;
  const int co0 = blockIdx.y * COB;
  const bool live = pix < npix;
  int n = 0, oy = 0, ox = 0;
  if (live) {
    n = (int)(pix / ((long long)a.Ho * a.Wo));
    const int rem = (int)(pix - (long long)n * a.Ho * a.Wo);
    oy = rem / a.Wo;
    ox = rem - oy * a.Wo;
  }
  int iy[3], ix[PX][3];
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    if (a.trans) {
      const int qy = oy + 1 - u;
      iy[u] = (qy >= 0 && qy % a.s == 0 && qy / a.s < a.Hi) ? qy / a.s : -1;
#pragma unroll
      for (int j = 0; j < PX; ++j) {
        const int qx = ox + j + 1 - u;
        ix[j][u] = (qx >= 0 && qx % a.s == 0 && qx / a.s < a.Wi) ? qx / a.s : -1;
      }
    } else {
      const int qy = a.s * oy + u - 1;
      iy[u] = (qy >= 0 && qy < a.Hi) ? qy : -1;
#pragma unroll
      for (int j = 0; j < PX; ++j) {
        const int qx = a.s * (ox + j) + u - 1;
        ix[j][u] = (qx >= 0 && qx < a.Wi) ? qx : -1;
      }
    }
  }
  float acc[PX][COB];
#pragma unroll
  for (int j = 0; j < PX; ++j)
#pragma unroll
    for (int k = 0; k < COB; ++k) acc[j][k] = 0.f;
  for (int c0 = 0; c0 < a.Ci; c0 += kCk) {
    const int ck = min(kCk, a.Ci - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < 9 * kCk * COB; i += kConvThreads) {
      const int k = i % COB, c = (i / COB) % kCk, t = i / (COB * kCk);
      float v = 0.f;
      if (c < ck && co0 + k < a.Co) v = a.w[(long long)(co0 + k) * a.sco + (long long)(c0 + c) * a.sci + t];
      ws[t][c][k] = v;
    }
    __syncthreads();
    if (!live) continue;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      if (iy[u] < 0) continue;
      const float* row = a.x + ((long long)n * a.Hi + iy[u]) * a.Wi * a.Ci + c0;
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        const int t = u * 3 + v;
        const float* px[PX];
#pragma unroll
        for (int j = 0; j < PX; ++j) px[j] = ix[j][v] >= 0 ? row + (long long)ix[j][v] * a.Ci : nullptr;
        if ((a.Ci & 3) == 0) {  // 16-byte input loads, 4 channels at a time
          for (int c = 0; c < ck; c += 4) {
            float4 x4[PX];
#pragma unroll
            for (int j = 0; j < PX; ++j)
              x4[j] = px[j] ? __ldg(reinterpret_cast<const float4*>(px[j] + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int cc = 0; cc < 4; ++cc)
#pragma unroll
              for (int k = 0; k < COB; ++k) {
                const float wk = ws[t][c + cc][k];
#pragma unroll
                for (int j = 0; j < PX; ++j) {
                  const float xv = cc == 0 ? x4[j].x : cc == 1 ? x4[j].y : cc == 2 ? x4[j].z : x4[j].w;
                  acc[j][k] = fmaf(xv, wk, acc[j][k]);
                }
              }
          }
        } else {
          for (int c = 0; c < ck; ++c) {
            float xv[PX];
#pragma unroll
            for (int j = 0; j < PX; ++j) xv[j] = px[j] ? __ldg(px[j] + c) : 0.f;
#pragma unroll
            for (int k = 0; k < COB; ++k) {
              const float wk = ws[t][c][k];
#pragma unroll
              for (int j = 0; j < PX; ++j) acc[j][k] = fmaf(xv[j], wk, acc[j][k]);
            }
          }
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int j = 0; j < PX; ++j) {
    float* py = a.y + (pix + j) * a.Co + co0;
#pragma unroll
    for (int k = 0; k < COB; ++k) {
      if (co0 + k >= a.Co) break;
      float v = acc[j][k];
      if (a.bias) v += a.bias[co0 + k];
      if (a.addend) v += a.addend[(pix + j) * a.Co + co0 + k];
      if (a.accumulate) v += py[k];
      py[k] = v;
    }
  }
}

// ------------------------------------------------------------------ weight gradient

// part[chunk][a][b][t] = sum_{pixels p of P in chunk} P[p, a] * Q[n, s o + (u, v) - 1, b]
struct TrWgrad {
  const float* P;
  int Hp, Wp, A;
  const float* Q;
  int Hq, Wq, Bc;
  int s, B;
  float* part;
  long long chunk;
};

// Tile AT x BT of (a, b) pairs x 9 taps; a thread owns 4 consecutive a for one b (36 accumulators).
// The 256 threads form KS = 256 / (AT BT / 4) groups that take interleaved 16-pixel slices of each
// staged row segment (split-K inside the block), folded in shared memory at the end in group order.
constexpr int kWgPx = 16;
constexpr int kWgSmem = 10240;  // floats of staging

// A block owns whole P rows; each round stages one SP-pixel row segment of P
// and the three Q rows it touches (s (SP - 1) + 3 columns) once, instead of 9 taps per pixel.  With
// stride 1 a thread slides a 3-column register window along the row (3 Q reads per pixel).
HS_DEV void cp_async4(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 4 : 0;  // src-size 0: the 4 bytes are zero-filled
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(n) : "memory");
}
HS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
HS_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int AT, int BT, int S>
struct WgCfg {
  static constexpr int TPG = AT * BT / 4;
  static constexpr int KS = 256 / TPG;
  static constexpr int SP = KS * kWgPx;
  static constexpr int QC = S * (SP - 1) + 3;
  static constexpr int STAGE = SP * AT + 3 * QC * BT;  // floats per buffer
  static constexpr int SMEM = 2 * STAGE * 4;           // double-buffered, bytes
};

// Rounds (row, SP-pixel segment) are staged with cp.async into two alternating buffers, so the
// next round's loads overlap this round's FMAs.
template <int AT, int BT, int S>
__global__ void __launch_bounds__(256, 2) k_tr_wgrad_rows(TrWgrad g) {
  using C = WgCfg<AT, BT, S>;
  constexpr int TPG = C::TPG, KS = C::KS, SP = C::SP, QC = C::QC;
  extern __shared__ __align__(16) float sm[];
  const int a0 = blockIdx.y * AT, b0 = blockIdx.z * BT;
  const int grp = threadIdx.x / TPG, lt = threadIdx.x % TPG;
  const int tb = lt % BT, ag = lt / BT;
  const long long nrows = (long long)g.B * g.Hp;
  const long long r0 = blockIdx.x * g.chunk, r1 = min(nrows, r0 + g.chunk);
  const int nseg = (g.Wp + SP - 1) / SP;
  const long long nround = (r1 > r0 ? r1 - r0 : 0) * nseg;
  auto issue = [&](long long k) {
    float* ps = sm + (k & 1) * C::STAGE;
    float* qs = ps + SP * AT;
    const long long row = r0 + k / nseg;
    const int x0 = (int)(k % nseg) * SP;
    const int npx = min(SP, g.Wp - x0);
    const int n = (int)(row / g.Hp), oy = (int)(row % g.Hp);
    for (int i = threadIdx.x; i < SP * AT; i += 256) {
      const int px = i / AT, ai = i % AT;
      const bool ok = px < npx && a0 + ai < g.A;
      cp_async4(ps + i, ok ? g.P + (row * g.Wp + x0 + px) * g.A + a0 + ai : g.P, ok);
    }
    for (int i = threadIdx.x; i < 3 * QC * BT; i += 256) {
      const int bi = i % BT, j = (i / BT) % QC, u = i / (QC * BT);
      const int qy = S * oy + u - 1, qx = S * x0 - 1 + j;
      const bool ok = j < S * (npx - 1) + 3 && qy >= 0 && qy < g.Hq && qx >= 0 && qx < g.Wq && b0 + bi < g.Bc;
      cp_async4(qs + i, ok ? g.Q + (((long long)n * g.Hq + qy) * g.Wq + qx) * g.Bc + b0 + bi : g.Q, ok);
    }
    cp_async_commit();
  };
  float acc[4][9];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int t = 0; t < 9; ++t) acc[i][t] = 0.f;
  if (nround > 0) issue(0);
  for (long long k = 0; k < nround; ++k) {
    if (k + 1 < nround) {
      issue(k + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    {
      const float* ps = sm + (k & 1) * C::STAGE;
      const float* qs = ps + SP * AT;
      const int pb = grp * kWgPx;
      if (S == 1) {
        float wa[3], wb[3];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          wa[u] = qs[(u * QC + pb) * BT + tb];
          wb[u] = qs[(u * QC + pb + 1) * BT + tb];
        }
#pragma unroll 4
        for (int kk = 0; kk < kWgPx; ++kk) {
          const float4 pa = *reinterpret_cast<const float4*>(ps + (pb + kk) * AT + 4 * ag);
#pragma unroll
          for (int u = 0; u < 3; ++u) {
            const float wc = qs[(u * QC + pb + kk + 2) * BT + tb];
            const float q3[3] = {wa[u], wb[u], wc};
#pragma unroll
            for (int v = 0; v < 3; ++v) {
              acc[0][u * 3 + v] = fmaf(pa.x, q3[v], acc[0][u * 3 + v]);
              acc[1][u * 3 + v] = fmaf(pa.y, q3[v], acc[1][u * 3 + v]);
              acc[2][u * 3 + v] = fmaf(pa.z, q3[v], acc[2][u * 3 + v]);
              acc[3][u * 3 + v] = fmaf(pa.w, q3[v], acc[3][u * 3 + v]);
            }
            wa[u] = wb[u];
            wb[u] = wc;
          }
        }
      } else {
#pragma unroll 2
        for (int kk = 0; kk < kWgPx; ++kk) {
          const float4 pa = *reinterpret_cast<const float4*>(ps + (pb + kk) * AT + 4 * ag);
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            const float q = qs[((t / 3) * QC + S * (pb + kk) + t % 3) * BT + tb];
            acc[0][t] = fmaf(pa.x, q, acc[0][t]);
            acc[1][t] = fmaf(pa.y, q, acc[1][t]);
            acc[2][t] = fmaf(pa.z, q, acc[2][t]);
            acc[3][t] = fmaf(pa.w, q, acc[3][t]);
          }
        }
      }
    }
    __syncthreads();  // this buffer is re-filled by round k + 2's issue
  }
  __syncthreads();
  if (grp > 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int t = 0; t < 9; ++t) sm[((grp - 1) * 36 + i * 9 + t) * TPG + lt] = acc[i][t];
  }
  __syncthreads();
  if (grp == 0) {
    for (int q = 1; q < KS; ++q)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int t = 0; t < 9; ++t) acc[i][t] += sm[((q - 1) * 36 + i * 9 + t) * TPG + lt];
    const int b = b0 + tb;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int a = a0 + 4 * ag + i;
      if (a < g.A && b < g.Bc) {
        float* out = g.part + (long long)blockIdx.x * g.A * g.Bc * 9 + ((long long)a * g.Bc + b) * 9;
#pragma unroll
        for (int t = 0; t < 9; ++t) out[t] = acc[i][t];
      }
    }
  }
}

// stage 1 of the partial sum: part2[grp][i] = sum of chunks [grp * per, (grp + 1) * per), in order
__global__ void k_tr_sum_parts1(const float* part, int nchunk, int per, long long n, float* part2) {
  const int grp = blockIdx.y;
  GRID_STRIDE(i, n) {
    double s = 0.0;
    const int c1 = min(nchunk, (grp + 1) * per);
    for (int c = grp * per; c < c1; ++c) s += part[(long long)c * n + i];
    part2[(long long)grp * n + i] = (float)s;
  }
}

// out[i] += sum_c part[c][i], chunks in order (deterministic)
__global__ void k_tr_sum_parts(const float* part, int nchunk, long long n, float* out) {
  GRID_STRIDE(i, n) {
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += part[(long long)c * n + i];
    out[i] += (float)s;
  }
}

// ------------------------------------------------------------------ per-channel reductions

enum ChanOp { kStats = 0, kBnBwd = 1, kSum = 2 };

struct TrChan {
  const float* z;
  const float* gy;
  long long M;
  int C;
  const float* mean;
  const float* inv;
  const float* gamma;
  const float* beta;
  int op;
  double* part;
  long long chunk;
};

HS_DEV float sigmoidf_(float a) { return 1.f / (1.f + __expf(-a)); }

// V consecutive channels per thread (float4 loads when C % 4 == 0), pixel lanes strided; double sums
template <int OP, int V>
__global__ void __launch_bounds__(256) k_tr_chan(TrChan a) {
  using VT = typename std::conditional<V == 4, float4, float>::type;
  __shared__ double sm[2][V][256];
  const int G = a.C / V;  // channel groups
  const int lanes = 256 / G;
  const int cg = threadIdx.x % G, lane = threadIdx.x / G;
  double q0[V], q1[V];
#pragma unroll
  for (int v = 0; v < V; ++v) q0[v] = q1[v] = 0.0;
  if (lane < lanes) {
    const long long p0 = blockIdx.x * a.chunk, p1 = min(a.M, p0 + a.chunk);
    float mu[V], iv[V], gm[V], bt[V];
    if (OP == kBnBwd) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        mu[v] = a.mean[cg * V + v];
        iv[v] = a.inv[cg * V + v];
        gm[v] = a.gamma[cg * V + v];
        bt[v] = a.beta[cg * V + v];
      }
    }
    const VT* zv = reinterpret_cast<const VT*>(a.z);
    const VT* gv = reinterpret_cast<const VT*>(a.gy);
#pragma unroll 4
    for (long long p = p0 + lane; p < p1; p += lanes) {
      const VT zz = zv[p * G + cg];
      const float* z = reinterpret_cast<const float*>(&zz);
      if (OP == kStats) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          q0[v] += z[v];
          q1[v] += (double)z[v] * z[v];
        }
      } else if (OP == kBnBwd) {
        const VT gg = gv[p * G + cg];
        const float* gy = reinterpret_cast<const float*>(&gg);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const float xh = (z[v] - mu[v]) * iv[v];
          const float ga = gy[v] * sigmoidf_(fmaf(gm[v], xh, bt[v]));
          q0[v] += ga;
          q1[v] += (double)ga * xh;
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) q0[v] += z[v];
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    sm[0][v][threadIdx.x] = q0[v];
    sm[1][v][threadIdx.x] = q1[v];
  }
  __syncthreads();
  if (threadIdx.x < a.C) {
    const int c = threadIdx.x, g = c / V, v = c % V;
    double s0 = 0.0, s1 = 0.0;
    for (int l = 0; l < lanes; ++l) {
      s0 += sm[0][v][l * G + g];
      s1 += sm[1][v][l * G + g];
    }
    a.part[((long long)blockIdx.x * a.C + c) * 2] = s0;
    a.part[((long long)blockIdx.x * a.C + c) * 2 + 1] = s1;
  }
}

struct TrChanFin {
  const double* part;
  int nchunk, C;
  long long M;
  int op;
  float* mean;  // kStats: batch mean / inv std out, running stats updated in place
  float* inv;
  float* rmean;
  float* rvar;
  float* g0;  // kBnBwd: dbeta (+=), kSum: the bias gradient (+=)
  float* g1;  // kBnBwd: dgamma (+=)
  float* s0;  // kBnBwd: sum(ga) / M, sum(ga xh) / M
  float* s1;
};

// one warp per channel: lanes take chunks lane, lane + 32, ... then a fixed shuffle tree (deterministic)
__global__ void k_tr_chan_fin(TrChanFin f) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= f.C) return;
  double q0 = 0.0, q1 = 0.0;
  for (int k = lane; k < f.nchunk; k += 32) {
    q0 += f.part[((long long)k * f.C + c) * 2];
    q1 += f.part[((long long)k * f.C + c) * 2 + 1];
  }
  q0 = warp_sum(q0);
  q1 = warp_sum(q1);
  if (lane) return;
  const double m = (double)f.M;
  if (f.op == kStats) {
    const double mean = q0 / m;
    const double var = fmax(q1 / m - mean * mean, 0.0);
    f.mean[c] = (float)mean;
    f.inv[c] = (float)(1.0 / sqrt(var + kBnEps));
    // autodiff.py:575-579: unbiased variance into the running buffer
    f.rmean[c] = (float)((1.0 - kMomentum) * f.rmean[c] + kMomentum * mean);
    f.rvar[c] = (float)((1.0 - kMomentum) * f.rvar[c] + kMomentum * var * (m / fmax(m - 1.0, 1.0)));
  } else if (f.op == kBnBwd) {
    f.g0[c] += (float)q0;
    f.g1[c] += (float)q1;
    f.s0[c] = (float)(q0 / m);
    f.s1[c] = (float)(q1 / m);
  } else {
    f.g0[c] += (float)q0;
  }
}

// ------------------------------------------------------------------ elementwise

// y = softplus(gamma (z - mean) inv + beta) (+ addend)
__global__ void k_tr_bn_act(const float* z, float* y, const float* addend, long long n, int C, const float* mean,
                            const float* inv, const float* gamma, const float* beta) {
  GRID_STRIDE(i, n) {
    const int c = (int)(i % C);
    const float a = fmaf(gamma[c], (z[i] - mean[c]) * inv[c], beta[c]);
    float v = fmaxf(a, 0.f) + log1pf(__expf(-fabsf(a)));
    if (addend) v += addend[i];
    y[i] = v;
  }
}

// gz = inv gamma (ga - mean(ga) - xh mean(ga xh)), ga = gy sigmoid(a)  (autodiff.py:582-590)
__global__ void k_tr_bn_dz(const float* z, const float* gy, float* gz, long long n, int C, const float* mean,
                           const float* inv, const float* gamma, const float* beta, const float* s0,
                           const float* s1) {
  GRID_STRIDE(i, n) {
    const int c = (int)(i % C);
    const float xh = (z[i] - mean[c]) * inv[c];
    const float ga = gy[i] * sigmoidf_(fmaf(gamma[c], xh, beta[c]));
    gz[i] = inv[c] * gamma[c] * (ga - s0[c] - xh * s1[c]);
  }
}

__global__ void k_tr_axpy(float* y, const float* x, long long n) {
  GRID_STRIDE(i, n) y[i] += x[i];
}

// media (n_models, 2, Ix, Iy) NCHW -> per-sample NHWC (B, Ix, Iy, 2)
__global__ void k_tr_media(const float* media, const int* model_of, float* out, int B, int ix, int iy) {
  const long long n = (long long)B * ix * iy * 2;
  GRID_STRIDE(i, n) {
    const int c = (int)(i & 1);
    const long long p = i >> 1;
    const int b = (int)(p / ((long long)ix * iy));
    const long long q = p - (long long)b * ix * iy;
    out[i] = media[((long long)model_of[b] * 2 + c) * ix * iy + q];
  }
}

// r (B, nx, ny) complex128 -> (B, Ix, Iy, 2) fp32 (the network reads r[:Ix, :Iy], ARCH.md)
__global__ void k_tr_r2(const double2* r, float* out, int B, int nx, int ny, int ix, int iy) {
  const long long n = (long long)B * ix * iy;
  GRID_STRIDE(p, n) {
    const int b = (int)(p / ((long long)ix * iy));
    const int q = (int)(p - (long long)b * ix * iy);
    const int i = q / iy, j = q - i * iy;
    const double2 v = r[((long long)b * nx + i) * ny + j];
    out[2 * p] = (float)v.x;
    out[2 * p + 1] = (float)v.y;
  }
}

// loss partials and the output gradient: u0 = s (out_0 + i out_1) on the network grid, 0 on the pad
__global__ void __launch_bounds__(256) k_tr_loss(const float* out, const double2* e, float* gout, int B, int nx,
                                                 int ny, int ix, int iy, double s, double* part) {
  __shared__ double scratch[2 * 9];
  const long long n = (long long)B * nx * ny;
  double acc[1] = {0.0};
  GRID_STRIDE(k, n) {
    const int b = (int)(k / ((long long)nx * ny));
    const int q = (int)(k - (long long)b * nx * ny);
    const int i = q / ny, j = q - i * ny;
    const double2 ev = e[k];
    double dr = -ev.x, di = -ev.y;
    if (i < ix && j < iy) {
      const long long p = ((long long)b * ix + i) * iy + j;
      dr += s * out[2 * p];
      di += s * out[2 * p + 1];
      gout[2 * p] = (float)(2.0 * s * dr / B);
      gout[2 * p + 1] = (float)(2.0 * s * di / B);
    }
    acc[0] += dr * dr + di * di;
  }
  block_sum<1>(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}

__global__ void k_tr_loss_fin(const double* part, int n, int B, double* loss) {
  if (threadIdx.x || blockIdx.x) return;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += part[i];
  *loss = s / B;
}

// ------------------------------------------------------------------ implicit layer (cuFFT)

// NHWC real (B, h, w, 2cc) -> complex (B, cc, 2h, 2w) zero-padded at the high end (pad2d_to)
__global__ void k_tr_pack_pad(const float* x, cufftComplex* z, int B, int h, int w, int cc) {
  const int H2 = 2 * h, W2 = 2 * w;
  const long long n = (long long)B * cc * H2 * W2;
  GRID_STRIDE(e, n) {
    const long long bk = e / ((long long)H2 * W2);
    const int b = (int)(bk / cc), k = (int)(bk - (long long)b * cc);
    const int rem = (int)(e - bk * H2 * W2);
    const int y = rem / W2, xx = rem - y * W2;
    cufftComplex v = make_float2(0.f, 0.f);
    if (y < h && xx < w) {
      const float* px = x + (((long long)b * h + y) * w + xx) * (2 * cc);
      v = make_float2(px[2 * k], px[2 * k + 1]);
    }
    z[e] = v;
  }
}

// out = in * (conj ? conj(S) : S), spectrum broadcast over the batch
__global__ void k_tr_spec_mul(const cufftComplex* in, cufftComplex* out, const cufftComplex* spec, long long per_b,
                              long long n, int conj) {
  GRID_STRIDE(e, n) {
    float2 s = spec[e % per_b];
    if (conj) s.y = -s.y;
    out[e] = cmul(in[e], s);
  }
}

// complex (B, cc, 2h, 2w) -> crop [:h, :w], / N, unpack to NHWC real; accumulate optionally
__global__ void k_tr_crop_unpack(const cufftComplex* z, float* x, int B, int h, int w, int cc, int accumulate) {
  const int H2 = 2 * h, W2 = 2 * w;
  const float inv = 1.f / (float)(H2 * W2);
  const long long n = (long long)B * h * w * cc;
  GRID_STRIDE(e, n) {
    const int k = (int)(e % cc);
    const long long pix = e / cc;
    const int b = (int)(pix / ((long long)h * w));
    const int q = (int)(pix - (long long)b * h * w);
    const int y = q / w, xx = q - y * w;
    const cufftComplex v = z[(((long long)b * cc + k) * H2 + y) * W2 + xx];
    float* px = x + pix * (2 * cc);
    if (accumulate) {
      px[2 * k] += v.x * inv;
      px[2 * k + 1] += v.y * inv;
    } else {
      px[2 * k] = v.x * inv;
      px[2 * k + 1] = v.y * inv;
    }
  }
}

// dS[k] = sum_b conj(X_b[k]) G_b[k] / N  (mul backward summed over the broadcast batch, ifft2 backward / N)
__global__ void k_tr_spec_grad(const cufftComplex* X, const cufftComplex* G, int B, long long per_b, double invN,
                               double2* dS) {
  GRID_STRIDE(k, per_b) {
    double2 s = make_double2(0.0, 0.0);
    for (int b = 0; b < B; ++b) s = zadd(s, zcmul(f2d(X[(long long)b * per_b + k]), f2d(G[(long long)b * per_b + k])));
    dS[k] = zscale(s, invN);
  }
}

// ------------------------------------------------------------------ Green spectrum and its gradient (complex128)

// place_kernel_corners (autodiff.py:323-337) of the float (re, im) kernel into (C, bh, bw)
__global__ void k_tr_green_embed(const float* kern, double2* kp, int C, int bh, int bw) {
  const long long n = (long long)C * bh * bw;
  GRID_STRIDE(e, n) {
    const int c = (int)(e / ((long long)bh * bw));
    const int rem = (int)(e - (long long)c * bh * bw);
    const int r = rem / bw, col = rem - r * bw;
    const int a = r == bh - 1 ? 0 : (r == 0 ? 1 : (r == 1 ? 2 : -1));
    const int q = col == bw - 1 ? 0 : (col == 0 ? 1 : (col == 1 ? 2 : -1));
    double2 v = make_double2(0.0, 0.0);
    if (a >= 0 && q >= 0) v = make_double2(kern[2 * (c * 9 + a * 3 + q)], kern[2 * (c * 9 + a * 3 + q) + 1]);
    kp[e] = v;
  }
}

// P dhat = conj(S) / (|S|^2 + eps) * (-1)^(u+v): the centred point source's spectrum on even grids
__global__ void k_tr_green_divide(const double2* S, double2* out, long long n, int bh, int bw) {
  GRID_STRIDE(e, n) {
    const int rem = (int)(e % ((long long)bh * bw));
    const int u = rem / bw, v = rem - u * bw;
    const double2 s = S[e];
    const double d = s.x * s.x + s.y * s.y + kSpecEps;
    const double sg = ((u + v) & 1) ? -1.0 : 1.0;
    out[e] = make_double2(sg * s.x / d, -sg * s.y / d);
  }
}

// crop the centred (gh, gw) window, ifftshift, 1/N of the inverse FFT
__global__ void k_tr_green_crop(const double2* R, double2* T, int C, int bh, int bw, int gh, int gw) {
  const long long n = (long long)C * gh * gw;
  const double inv = 1.0 / ((double)bh * bw);
  const int oy = bh / 2 - gh / 2, ox = bw / 2 - gw / 2;
  GRID_STRIDE(e, n) {
    const int c = (int)(e / ((long long)gh * gw));
    const int rem = (int)(e - (long long)c * gh * gw);
    const int r = rem / gw, col = rem - r * gw;
    const int sr = (r + gh / 2) % gh, sc = (col + gw / 2) % gw;
    T[e] = zscale(R[((long long)c * bh + oy + sr) * bw + ox + sc], inv);
  }
}

__global__ void k_tr_to_c64(const double2* in, cufftComplex* out, long long n) {
  GRID_STRIDE(e, n) out[e] = make_float2((float)in[e].x, (float)in[e].y);
}

// backward of crop + ifftshift: gR (C, bh, bw) = 0 except the window, gR[oy + r] = gU[(r - g/2) mod g]
__global__ void k_tr_gb_embed(const double2* gU, double2* gR, int C, int bh, int bw, int gh, int gw) {
  const long long n = (long long)C * bh * bw;
  const int oy = bh / 2 - gh / 2, ox = bw / 2 - gw / 2;
  GRID_STRIDE(e, n) {
    const int c = (int)(e / ((long long)bh * bw));
    const int rem = (int)(e - (long long)c * bh * bw);
    const int r = rem / bw - oy, col = rem % bw - ox;
    double2 v = make_double2(0.0, 0.0);
    if (r >= 0 && r < gh && col >= 0 && col < gw) {
      const int sr = ((r - gh / 2) % gh + gh) % gh, sc = ((col - gw / 2) % gw + gw) % gw;
      v = gU[((long long)c * gh + sr) * gw + sc];
    }
    gR[e] = v;
  }
}

// gQ = fft2(gR) / N; gP = gQ conj(dhat); gS = conj(gP) eps / D^2 - gP S^2 / D^2 (Wirtinger chain
// through conj / mul / add / div of green.py:73-75 in the convention of autodiff.py:3-12)
__global__ void k_tr_gb_divide(double2* g, const double2* S, long long n, int bh, int bw) {
  const double invN = 1.0 / ((double)bh * bw);
  GRID_STRIDE(e, n) {
    const int rem = (int)(e % ((long long)bh * bw));
    const int u = rem / bw, v = rem - u * bw;
    const double sg = ((u + v) & 1) ? -invN : invN;
    const double2 gp = zscale(g[e], sg);
    const double2 s = S[e];
    const double d = s.x * s.x + s.y * s.y + kSpecEps;
    const double id2 = 1.0 / (d * d);
    const double2 s2 = make_double2(s.x * s.x - s.y * s.y, 2.0 * s.x * s.y);
    const double2 t = zmul(gp, s2);
    g[e] = make_double2((gp.x * kSpecEps - t.x) * id2, (-gp.y * kSpecEps - t.y) * id2);
  }
}

// place_kernel_corners backward: gather the 9 embedded positions into the kernel gradient (+=)
__global__ void k_tr_gb_gather(const double2* gkp, float* gk, int C, int bh, int bw) {
  const int n = C * 9;
  GRID_STRIDE(e, n) {
    const int c = (int)(e / 9), t = (int)(e % 9);
    const int a = t / 3, q = t % 3;
    const int r = a == 0 ? bh - 1 : a - 1, col = q == 0 ? bw - 1 : q - 1;
    const double2 v = gkp[((long long)c * bh + r) * bw + col];
    gk[2 * e] += (float)v.x;
    gk[2 * e + 1] += (float)v.y;
  }
}

// ------------------------------------------------------------------ Adam (torch.optim.Adam defaults)

__global__ void k_tr_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1, float b2,
                          float eps, float c1, float c2) {
  GRID_STRIDE(i, n) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}

// ------------------------------------------------------------------ weight re-packing

// dst[o][u][v][i] = src[o][i][u'][v'] (src_io = 0) or src[i][o][u'][v'] (src_io = 1), (u', v') = flip ? (2-u, 2-v) : (u, v)
struct Repack {
  const float* src;
  float* dst;
  int O, I, src_io, flip;
};

__global__ void k_tr_repack(const Repack* tab) {
  const Repack r = tab[blockIdx.y];
  const int n = r.O * r.I * 9;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int i = e % r.I, t = (e / r.I) % 9, o = e / (9 * r.I);
    const int ts = r.flip ? 8 - t : t;
    r.dst[e] = r.src_io ? r.src[((long long)i * r.O + o) * 9 + ts] : r.src[((long long)o * r.I + i) * 9 + ts];
  }
}

// ------------------------------------------------------------------ the trainer

enum Kind { kS1 = 0, kS2 = 1, kT2 = 2 };

struct LayerP {
  size_t w = 0, b = 0, gamma = 0, beta = 0, mean = 0, var = 0;
  int cin = 0, cout = 0, kind = 0;  // kind: kS1 / kS2 / kT2
  bool bn = false, transposed = false;
  float* wf = nullptr;  // forward weights in the tensor-core layout [out][ky][kx][in] (re-packed per step)
  float* wd = nullptr;  // data-gradient weights, same layout
  float* st_mean = nullptr;  // batch statistics of the current step
  float* st_inv = nullptr;
};

struct Lvl {  // one level's saved activations (NHWC) and gradients
  float *z = nullptr, *c = nullptr, *gc = nullptr, *za = nullptr, *t = nullptr, *o = nullptr, *go = nullptr;
};

}  // namespace
}  // namespace hs

struct hs_trainer {
  hs_train_desc_t d{};
  int L = 0, ix = 0, iy = 0, B = 0, hc = 0, wc = 0, cc = 0;
  size_t nparam = 0;
  float *P = nullptr, *G = nullptr, *M = nullptr, *V = nullptr;
  int t = 0;
  hs::LayerP enc_stem, sol_stem, head;
  hs::LayerP enc_a[8], enc_b[8], enc_down[8], sol_a[8], sol_b[8], sol_down[8], up[8], ures_a[8], ures_b[8];
  size_t implicit = 0;
  hs::Lvl E[8], S[8], U[8];
  float *media_b = nullptr, *r2 = nullptr, *imp = nullptr, *gimp = nullptr, *out = nullptr, *gout = nullptr;
  float *scr_t = nullptr, *scr_z = nullptr, *s0 = nullptr, *s1 = nullptr;
  double* chan_part = nullptr;
  long long chan_part_cap = 0;
  float* wg_part = nullptr;
  long long wg_part_cap = 0;
  double *loss_part = nullptr, *loss_dev = nullptr;
  int* model_dev = nullptr;
  hs::Repack* repack = nullptr;  // device table, one entry per packed weight array
  int n_repack = 0;
  float* zero_bias = nullptr;
  cufftComplex *Xf = nullptr, *Yb = nullptr, *spec = nullptr;
  double2 *big1 = nullptr, *big2 = nullptr, *gG = nullptr;
  cufftHandle pB = 0, p1 = 0, p2 = 0;
  bool plans = false;
  std::vector<void*> allocs;
  char* grad_arena = nullptr;
  size_t grad_arena_bytes = 0;
  ~hs_trainer() {
    for (void* p : allocs) cudaFree(p);
    if (plans) {
      cufftDestroy(pB);
      cufftDestroy(p1);
      cufftDestroy(p2);
    }
  }
};

namespace hs {
namespace {

// walk netparams.param_spec (netparams.py:31-53): the same order and sizes
struct Spec {
  size_t off = 0;
  LayerP conv(int co, int ci, int kind, bool bn = true) {
    LayerP p;
    p.cin = ci;
    p.cout = co;
    p.kind = kind;
    p.transposed = kind == kT2;
    p.bn = bn;
    p.w = off;
    off += (size_t)co * ci * 9;
    p.b = off;
    off += co;
    if (bn) {
      p.gamma = off;
      p.beta = off + co;
      p.mean = off + 2 * co;
      p.var = off + 3 * co;
      off += 4 * (size_t)co;
    }
    return p;
  }
};

void build_layout(hs_trainer* t) {
  Spec s;
  const int* C = t->d.channels;
  const int L = t->L;
  for (int side = 0; side < 2; ++side) {
    LayerP* stem = side ? &t->sol_stem : &t->enc_stem;
    LayerP* la = side ? t->sol_a : t->enc_a;
    LayerP* lb = side ? t->sol_b : t->enc_b;
    LayerP* ld = side ? t->sol_down : t->enc_down;
    *stem = s.conv(C[0], 2, kS1);
    la[0] = s.conv(C[0], C[0], kS1);
    lb[0] = s.conv(C[0], C[0], kS1, false);
    for (int lv = 1; lv < L; ++lv) {
      ld[lv] = s.conv(C[lv], C[lv - 1], kS2);
      la[lv] = s.conv(C[lv], C[lv], kS1);
      lb[lv] = s.conv(C[lv], C[lv], kS1, false);
    }
  }
  t->implicit = s.off;
  s.off += (size_t)(C[L - 1] / 2) * 9 * 2;
  for (int lv = L - 1; lv >= 1; --lv) {
    t->up[lv] = s.conv(C[lv - 1], C[lv], kT2);
    t->ures_a[lv] = s.conv(C[lv - 1], C[lv - 1], kS1);
    t->ures_b[lv] = s.conv(C[lv - 1], C[lv - 1], kS1, false);
  }
  t->head = s.conv(2, C[0], kS1, false);
  t->nparam = s.off;
}

template <class T>
T* dalloc(hs_trainer* t, size_t count) {
  void* p = nullptr;
  if (cudaMalloc(&p, count * sizeof(T) + 16) != cudaSuccess) return nullptr;
  t->allocs.push_back(p);
  return static_cast<T*>(p);
}

// ----------------------------------------------------------------- launch helpers

void conv_launch(const float* x, int Hi, int Wi, int Ci, float* y, int Ho, int Wo, int Co, const float* w, int sco,
                 int sci, const float* bias, const float* addend, int trans, int s, int accumulate, int B,
                 cudaStream_t st) {
  TrConv a{x, Hi, Wi, Ci, y, Ho, Wo, Co, w, sco, sci, bias, addend, trans, s, accumulate, B};
  const long long npix = (long long)B * Ho * Wo;
  if (Wo % 4 == 0) {
    const unsigned gx = (unsigned)((npix / 4 + kConvThreads - 1) / kConvThreads);
    if (Co >= 16) k_tr_conv<16, 4><<<dim3(gx, (Co + 15) / 16), kConvThreads, 0, st>>>(a);
    else if (Co >= 8) k_tr_conv<8, 4><<<dim3(gx, (Co + 7) / 8), kConvThreads, 0, st>>>(a);
    else if (Co >= 4) k_tr_conv<4, 4><<<dim3(gx, (Co + 3) / 4), kConvThreads, 0, st>>>(a);
    else k_tr_conv<2, 4><<<dim3(gx, (Co + 1) / 2), kConvThreads, 0, st>>>(a);
  } else {
    const unsigned gx = (unsigned)((npix + kConvThreads - 1) / kConvThreads);
    if (Co >= 16) k_tr_conv<16, 1><<<dim3(gx, (Co + 15) / 16), kConvThreads, 0, st>>>(a);
    else if (Co >= 8) k_tr_conv<8, 1><<<dim3(gx, (Co + 7) / 8), kConvThreads, 0, st>>>(a);
    else if (Co >= 4) k_tr_conv<4, 1><<<dim3(gx, (Co + 3) / 4), kConvThreads, 0, st>>>(a);
    else k_tr_conv<2, 1><<<dim3(gx, (Co + 1) / 2), kConvThreads, 0, st>>>(a);
  }
  prof::count(1);
}

template <int AT, int BT, int S>
void launch_wg(dim3 grid, const TrWgrad& g, cudaStream_t st) {
  using C = WgCfg<AT, BT, S>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tr_wgrad_rows<AT, BT, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  k_tr_wgrad_rows<AT, BT, S><<<grid, 256, C::SMEM, st>>>(g);
}

void wgrad_launch(hs_trainer* t, const float* P, int Hp, int Wp, int A, const float* Q, int Hq, int Wq, int Bc, int s,
                  float* out, cudaStream_t st) {
  const long long nrows = (long long)t->B * Hp;
  const int AT = A >= 32 ? 32 : 16, BT = Bc >= 32 ? 32 : 16;
  const int tiles = ((A + AT - 1) / AT) * ((Bc + BT - 1) / BT);
  const long long per = (long long)A * Bc * 9;
  long long nchunk = (3 * 148 + tiles - 1) / tiles;
  nchunk = std::min(nchunk, nrows);
  nchunk = std::min(nchunk, std::max(1LL, t->wg_part_cap / (2 * per)));
  const long long chunk = (nrows + nchunk - 1) / nchunk;  // rows per block
  nchunk = (nrows + chunk - 1) / chunk;
  TrWgrad g{P, Hp, Wp, A, Q, Hq, Wq, Bc, s, t->B, t->wg_part, chunk};
  const int slot = prof::start(prof::TRAIN_WGRAD, st);
  const dim3 grid((unsigned)nchunk, (A + AT - 1) / AT, (Bc + BT - 1) / BT);
#define HS_WG(ATV, BTV)                                                                       \
  if (AT == ATV && BT == BTV) {                                                               \
    if (s == 1) launch_wg<ATV, BTV, 1>(grid, g, st);                                          \
    else launch_wg<ATV, BTV, 2>(grid, g, st);                                                 \
  }
  HS_WG(16, 16)
  HS_WG(16, 32)
  HS_WG(32, 16)
  HS_WG(32, 32)
#undef HS_WG
  // deterministic two-stage sum of the chunk partials
  const int per_grp = 16;
  const int ngrp = (int)((nchunk + per_grp - 1) / per_grp);
  float* part2 = t->wg_part + nchunk * per;
  k_tr_sum_parts1<<<dim3(g1(per), ngrp), 256, 0, st>>>(t->wg_part, (int)nchunk, per_grp, per, part2);
  k_tr_sum_parts<<<g1(per), 256, 0, st>>>(part2, ngrp, per, out);
  prof::stop(slot, st, 18.0 * (double)nrows * Wp * A * Bc);
  prof::count(3);
}

// per-channel reduction + finalisation over an NHWC tensor of M pixels
void chan_launch(hs_trainer* t, int op, const float* z, const float* gy, long long M, int C, const LayerP* p,
                 float* g0, float* g1_, cudaStream_t st) {
  long long nchunk = std::min<long long>(4 * 148, std::max(1LL, M / 256));
  nchunk = std::min(nchunk, t->chan_part_cap / (2LL * C));
  const long long chunk = (M + nchunk - 1) / nchunk;
  nchunk = (M + chunk - 1) / chunk;
  TrChan a{z, gy, M, C, nullptr, nullptr, nullptr, nullptr, op, t->chan_part, chunk};
  if (op == kBnBwd) {
    a.mean = p->st_mean;
    a.inv = p->st_inv;
    a.gamma = t->P + p->gamma;
    a.beta = t->P + p->beta;
  }
#define HS_CH(OPV)                                                                          \
  if (op == OPV) {                                                                          \
    if (C % 4 == 0) k_tr_chan<OPV, 4><<<(unsigned)nchunk, 256, 0, st>>>(a);               \
    else k_tr_chan<OPV, 1><<<(unsigned)nchunk, 256, 0, st>>>(a);                          \
  }
  HS_CH(kStats)
  HS_CH(kBnBwd)
  HS_CH(kSum)
#undef HS_CH
  TrChanFin f{t->chan_part, (int)nchunk, C, M, op, nullptr, nullptr, nullptr, nullptr, g0, g1_, t->s0, t->s1};
  if (op == kStats) {
    f.mean = p->st_mean;
    f.inv = p->st_inv;
    f.rmean = t->P + p->mean;
    f.rvar = t->P + p->var;
  }
  k_tr_chan_fin<<<(C + 7) / 8, 256, 0, st>>>(f);
  prof::count(2);
}


// forward convolution of layer p (conv stride 1/2 or transposed stride 2) into y (+ bias, + addend):
// the tcgen05 implicit-GEMM kernel (conv_tc.cu, exact bf16x3 split) where the shape has one, else SIMT
void conv_fwd(hs_trainer* t, const LayerP& p, int kind, const float* x, int Hi, int Wi, float* y, int Ho, int Wo,
              const float* addend, cudaStream_t st) {
  const float* w = t->P + p.w;
  const int s = kind == kS1 ? 1 : 2, tr = kind == kT2;
  const double flops = 18.0 * t->B * (tr ? (double)Hi * Wi : (double)Ho * Wo) * p.cin * p.cout;
  struct Scope {
    int slot;
    cudaStream_t st;
    double w;
    ~Scope() { prof::stop(slot, st, w); }
  } scope{prof::start(prof::CONV, st), st, flops};
  if (p.wf && conv_tc_supported(p.cin, p.cout, s, tr, Hi, Wi, Wo) &&
      conv_tc_launch(x, Hi, Wi, p.cin, y, Ho, Wo, p.cout, s, tr, p.wf, t->P + p.b, 0, addend,
                     (long long)Ho * Wo * p.cout, 0, nullptr, nullptr, nullptr, t->B, st)) {
    prof::count(1);
    return;
  }
  if (kind == kT2)
    conv_launch(x, Hi, Wi, p.cin, y, Ho, Wo, p.cout, w, 9, p.cout * 9, t->P + p.b, addend, 1, 2, 0, t->B, st);
  else
    conv_launch(x, Hi, Wi, p.cin, y, Ho, Wo, p.cout, w, p.cin * 9, 9, t->P + p.b, addend, 0, s, 0, t->B, st);
}

// gx += data gradient: a stride-1 conv with flipped, transposed weights (conv s1), a transposed conv
// (conv s2) or a stride-2 conv (transposed conv) -- on the tensor cores where the shape allows
void dgrad(hs_trainer* t, const LayerP& p, int kind, const float* gz, int Ho, int Wo, float* gx, int Hi, int Wi,
           cudaStream_t st) {
  const float* w = t->P + p.w;
  const int s = kind == kS1 ? 1 : 2;
  const double flops = 18.0 * t->B * (kind == kT2 ? (double)Hi * Wi : (double)Ho * Wo) * p.cin * p.cout;
  struct Scope {
    int slot;
    cudaStream_t st;
    double w;
    ~Scope() { prof::stop(slot, st, w); }
  } scope{prof::start(prof::CONV, st), st, flops};
  // the adjoint's own shape: in = p.cout at (Ho, Wo), out = p.cin at (Hi, Wi); conv s1 -> conv s1,
  // conv s2 -> transposed conv, transposed conv -> conv s2
  const int astride = s, atr = kind == kS2;
  if (p.wd && conv_tc_supported(p.cout, p.cin, astride, atr, Ho, Wo, Wi) &&
      conv_tc_launch(gz, Ho, Wo, p.cout, gx, Hi, Wi, p.cin, astride, atr, p.wd, t->zero_bias, 0, nullptr, 0, 0,
                     nullptr, gx, nullptr, t->B, st)) {
    prof::count(1);
    return;
  }
  if (kind == kT2)
    conv_launch(gz, Ho, Wo, p.cout, gx, Hi, Wi, p.cin, w, p.cout * 9, 9, nullptr, nullptr, 0, 2, 1, t->B, st);
  else
    conv_launch(gz, Ho, Wo, p.cout, gx, Hi, Wi, p.cin, w, 9, p.cin * 9, nullptr, nullptr, 1, s, 1, t->B, st);
}

// backward of conv_fwd given the complete output gradient gz: weight / bias gradients (+=), gx (+=) if wanted
void conv_bwd(hs_trainer* t, const LayerP& p, int kind, const float* x, int Hi, int Wi, const float* gz, int Ho,
              int Wo, float* gx, cudaStream_t st) {
  chan_launch(t, kSum, gz, nullptr, (long long)t->B * Ho * Wo, p.cout, &p, t->G + p.b, nullptr, st);
  if (kind == kT2)
    wgrad_launch(t, x, Hi, Wi, p.cin, gz, Ho, Wo, p.cout, 2, t->G + p.w, st);
  else
    wgrad_launch(t, gz, Ho, Wo, p.cout, x, Hi, Wi, p.cin, kind == kS2 ? 2 : 1, t->G + p.w, st);
  if (gx) dgrad(t, p, kind, gz, Ho, Wo, gx, Hi, Wi, st);
}

// y = softplus(BN_train(conv(x) + b)) (+ addend); z keeps the pre-BN output
void cbs_fwd(hs_trainer* t, const LayerP& p, int kind, const float* x, int Hi, int Wi, float* z, float* y, int Ho,
             int Wo, const float* addend, cudaStream_t st) {
  conv_fwd(t, p, kind, x, Hi, Wi, z, Ho, Wo, nullptr, st);
  const long long M = (long long)t->B * Ho * Wo;
  chan_launch(t, kStats, z, nullptr, M, p.cout, &p, nullptr, nullptr, st);
  k_tr_bn_act<<<g1(M * p.cout), 256, 0, st>>>(z, y, addend, M * p.cout, p.cout, p.st_mean, p.st_inv,
                                               t->P + p.gamma, t->P + p.beta);
  prof::count(1);
}

void cbs_bwd(hs_trainer* t, const LayerP& p, int kind, const float* x, int Hi, int Wi, const float* z,
             const float* gy, int Ho, int Wo, float* gx, cudaStream_t st) {
  const long long M = (long long)t->B * Ho * Wo;
  chan_launch(t, kBnBwd, z, gy, M, p.cout, &p, t->G + p.beta, t->G + p.gamma, st);
  k_tr_bn_dz<<<g1(M * p.cout), 256, 0, st>>>(z, gy, t->scr_z, M * p.cout, p.cout, p.st_mean, p.st_inv,
                                              t->P + p.gamma, t->P + p.beta, t->s0, t->s1);
  prof::count(1);
  conv_bwd(t, p, kind, x, Hi, Wi, t->scr_z, Ho, Wo, gx, st);
}

// y = x + conv_b(cbs_a(x)) + b_b
void res_fwd(hs_trainer* t, const LayerP& a, const LayerP& b, const float* x, int H, int W, float* za, float* tt,
             float* y, cudaStream_t st) {
  cbs_fwd(t, a, kS1, x, H, W, za, tt, H, W, nullptr, st);
  conv_fwd(t, b, kS1, tt, H, W, y, H, W, x, st);
}

void res_bwd(hs_trainer* t, const LayerP& a, const LayerP& b, const float* x, int H, int W, const float* za,
             const float* tt, const float* gy, float* gx, cudaStream_t st) {
  const long long n = (long long)t->B * H * W * a.cout;
  cudaMemsetAsync(t->scr_t, 0, n * sizeof(float), st);
  conv_bwd(t, b, kS1, tt, H, W, gy, H, W, t->scr_t, st);
  cbs_bwd(t, a, kS1, x, H, W, za, t->scr_t, H, W, gx, st);
  k_tr_axpy<<<g1(n), 256, 0, st>>>(gx, gy, n);
  prof::count(1);
}

int fft_check(cufftResult r) { return r == CUFFT_SUCCESS ? HS_OK : HS_ECUDA; }

// Green spectrum of the current kernel weights (complex128 chain, stored complex64); keeps S in big1
int green_fwd(hs_trainer* t, cudaStream_t st) {
  const int C = t->cc, gh = 2 * t->hc, gw = 2 * t->wc, bh = 3 * gh, bw = 3 * gw;
  const long long nb = (long long)C * bh * bw, ng = (long long)C * gh * gw;
  k_tr_green_embed<<<g1(nb), 256, 0, st>>>(t->P + t->implicit, t->big1, C, bh, bw);
  if (fft_check(cufftExecZ2Z(t->p1, t->big1, t->big1, CUFFT_FORWARD))) return HS_ECUDA;
  k_tr_green_divide<<<g1(nb), 256, 0, st>>>(t->big1, t->big2, nb, bh, bw);
  if (fft_check(cufftExecZ2Z(t->p1, t->big2, t->big2, CUFFT_INVERSE))) return HS_ECUDA;
  k_tr_green_crop<<<g1(ng), 256, 0, st>>>(t->big2, t->gG, C, bh, bw, gh, gw);
  if (fft_check(cufftExecZ2Z(t->p2, t->gG, t->gG, CUFFT_FORWARD))) return HS_ECUDA;
  k_tr_to_c64<<<g1(ng), 256, 0, st>>>(t->gG, t->spec, ng);
  prof::count(4);
  return HS_OK;
}

// kernel-weight gradient from dS (in gG, complex128)
int green_bwd(hs_trainer* t, cudaStream_t st) {
  const int C = t->cc, gh = 2 * t->hc, gw = 2 * t->wc, bh = 3 * gh, bw = 3 * gw;
  const long long nb = (long long)C * bh * bw;
  if (fft_check(cufftExecZ2Z(t->p2, t->gG, t->gG, CUFFT_INVERSE))) return HS_ECUDA;  // N ifft2
  k_tr_gb_embed<<<g1(nb), 256, 0, st>>>(t->gG, t->big2, C, bh, bw, gh, gw);
  if (fft_check(cufftExecZ2Z(t->p1, t->big2, t->big2, CUFFT_FORWARD))) return HS_ECUDA;
  k_tr_gb_divide<<<g1(nb), 256, 0, st>>>(t->big2, t->big1, nb, bh, bw);
  if (fft_check(cufftExecZ2Z(t->p1, t->big2, t->big2, CUFFT_INVERSE))) return HS_ECUDA;  // N ifft2
  k_tr_gb_gather<<<1, 256, 0, st>>>(t->big2, t->G + t->implicit, C, bh, bw);
  prof::count(3);
  return HS_OK;
}

int implicit_fwd(hs_trainer* t, const float* x, float* y, cudaStream_t st) {
  const long long per_b = (long long)t->cc * 4 * t->hc * t->wc, n = t->B * per_b;
  k_tr_pack_pad<<<g1(n), 256, 0, st>>>(x, t->Xf, t->B, t->hc, t->wc, t->cc);
  if (fft_check(cufftExecC2C(t->pB, t->Xf, t->Xf, CUFFT_FORWARD))) return HS_ECUDA;
  k_tr_spec_mul<<<g1(n), 256, 0, st>>>(t->Xf, t->Yb, t->spec, per_b, n, 0);
  if (fft_check(cufftExecC2C(t->pB, t->Yb, t->Yb, CUFFT_INVERSE))) return HS_ECUDA;
  k_tr_crop_unpack<<<g1((long long)t->B * t->hc * t->wc * t->cc), 256, 0, st>>>(t->Yb, y, t->B, t->hc, t->wc, t->cc,
                                                                                 0);
  prof::count(3);
  return HS_OK;
}

int implicit_bwd(hs_trainer* t, const float* gy, float* gx, cudaStream_t st) {
  const long long per_b = (long long)t->cc * 4 * t->hc * t->wc, n = t->B * per_b;
  k_tr_pack_pad<<<g1(n), 256, 0, st>>>(gy, t->Yb, t->B, t->hc, t->wc, t->cc);
  if (fft_check(cufftExecC2C(t->pB, t->Yb, t->Yb, CUFFT_FORWARD))) return HS_ECUDA;
  k_tr_spec_grad<<<g1(per_b), 256, 0, st>>>(t->Xf, t->Yb, t->B, per_b, 1.0 / (4.0 * t->hc * t->wc), t->gG);
  k_tr_spec_mul<<<g1(n), 256, 0, st>>>(t->Yb, t->Yb, t->spec, per_b, n, 1);
  if (fft_check(cufftExecC2C(t->pB, t->Yb, t->Yb, CUFFT_INVERSE))) return HS_ECUDA;
  k_tr_crop_unpack<<<g1((long long)t->B * t->hc * t->wc * t->cc), 256, 0, st>>>(t->Yb, gx, t->B, t->hc, t->wc, t->cc,
                                                                                 1);
  prof::count(4);
  return green_bwd(t, st);
}

int forward(hs_trainer* t, cudaStream_t st) {
  const int L = t->L;
  auto H = [&](int l) { return t->ix >> l; };
  auto W = [&](int l) { return t->iy >> l; };
  // encoder
  cbs_fwd(t, t->enc_stem, kS1, t->media_b, H(0), W(0), t->E[0].z, t->E[0].c, H(0), W(0), nullptr, st);
  res_fwd(t, t->enc_a[0], t->enc_b[0], t->E[0].c, H(0), W(0), t->E[0].za, t->E[0].t, t->E[0].o, st);
  for (int l = 1; l < L; ++l) {
    cbs_fwd(t, t->enc_down[l], kS2, t->E[l - 1].o, H(l - 1), W(l - 1), t->E[l].z, t->E[l].c, H(l), W(l), nullptr, st);
    res_fwd(t, t->enc_a[l], t->enc_b[l], t->E[l].c, H(l), W(l), t->E[l].za, t->E[l].t, t->E[l].o, st);
  }
  // solver down path
  cbs_fwd(t, t->sol_stem, kS1, t->r2, H(0), W(0), t->S[0].z, t->S[0].c, H(0), W(0), t->E[0].o, st);
  res_fwd(t, t->sol_a[0], t->sol_b[0], t->S[0].c, H(0), W(0), t->S[0].za, t->S[0].t, t->S[0].o, st);
  for (int l = 1; l < L; ++l) {
    cbs_fwd(t, t->sol_down[l], kS2, t->S[l - 1].o, H(l - 1), W(l - 1), t->S[l].z, t->S[l].c, H(l), W(l), t->E[l].o,
            st);
    res_fwd(t, t->sol_a[l], t->sol_b[l], t->S[l].c, H(l), W(l), t->S[l].za, t->S[l].t, t->S[l].o, st);
  }
  int rc = implicit_fwd(t, t->S[L - 1].o, t->imp, st);
  if (rc) return rc;
  // up path: U[l] lives at level l-1
  for (int l = L - 1; l >= 1; --l) {
    const float* x = l == L - 1 ? t->imp : t->U[l + 1].o;
    cbs_fwd(t, t->up[l], kT2, x, H(l), W(l), t->U[l].z, t->U[l].c, H(l - 1), W(l - 1), t->S[l - 1].o, st);
    res_fwd(t, t->ures_a[l], t->ures_b[l], t->U[l].c, H(l - 1), W(l - 1), t->U[l].za, t->U[l].t, t->U[l].o, st);
  }
  conv_fwd(t, t->head, kS1, t->U[1].o, H(0), W(0), t->out, H(0), W(0), nullptr, st);
  return HS_OK;
}

int backward(hs_trainer* t, cudaStream_t st) {
  const int L = t->L;
  auto H = [&](int l) { return t->ix >> l; };
  auto W = [&](int l) { return t->iy >> l; };
  conv_bwd(t, t->head, kS1, t->U[1].o, H(0), W(0), t->gout, H(0), W(0), t->U[1].go, st);
  for (int l = 1; l < L; ++l) {
    const long long n = (long long)t->B * H(l - 1) * W(l - 1) * t->d.channels[l - 1];
    res_bwd(t, t->ures_a[l], t->ures_b[l], t->U[l].c, H(l - 1), W(l - 1), t->U[l].za, t->U[l].t, t->U[l].go,
            t->U[l].gc, st);
    k_tr_axpy<<<g1(n), 256, 0, st>>>(t->S[l - 1].go, t->U[l].gc, n);  // the skip connection
    prof::count(1);
    const float* x = l == L - 1 ? t->imp : t->U[l + 1].o;
    float* gx = l == L - 1 ? t->gimp : t->U[l + 1].go;
    cbs_bwd(t, t->up[l], kT2, x, H(l), W(l), t->U[l].z, t->U[l].gc, H(l - 1), W(l - 1), gx, st);
  }
  int rc = implicit_bwd(t, t->gimp, t->S[L - 1].go, st);
  if (rc) return rc;
  for (int l = L - 1; l >= 1; --l) {
    const long long n = (long long)t->B * H(l) * W(l) * t->d.channels[l];
    res_bwd(t, t->sol_a[l], t->sol_b[l], t->S[l].c, H(l), W(l), t->S[l].za, t->S[l].t, t->S[l].go, t->S[l].gc, st);
    k_tr_axpy<<<g1(n), 256, 0, st>>>(t->E[l].go, t->S[l].gc, n);  // + e_l
    prof::count(1);
    cbs_bwd(t, t->sol_down[l], kS2, t->S[l - 1].o, H(l - 1), W(l - 1), t->S[l].z, t->S[l].gc, H(l), W(l),
            t->S[l - 1].go, st);
  }
  {
    const long long n = (long long)t->B * H(0) * W(0) * t->d.channels[0];
    res_bwd(t, t->sol_a[0], t->sol_b[0], t->S[0].c, H(0), W(0), t->S[0].za, t->S[0].t, t->S[0].go, t->S[0].gc, st);
    k_tr_axpy<<<g1(n), 256, 0, st>>>(t->E[0].go, t->S[0].gc, n);
    prof::count(1);
    cbs_bwd(t, t->sol_stem, kS1, t->r2, H(0), W(0), t->S[0].z, t->S[0].gc, H(0), W(0), nullptr, st);
  }
  for (int l = L - 1; l >= 1; --l) {
    res_bwd(t, t->enc_a[l], t->enc_b[l], t->E[l].c, H(l), W(l), t->E[l].za, t->E[l].t, t->E[l].go, t->E[l].gc, st);
    cbs_bwd(t, t->enc_down[l], kS2, t->E[l - 1].o, H(l - 1), W(l - 1), t->E[l].z, t->E[l].gc, H(l), W(l),
            t->E[l - 1].go, st);
  }
  res_bwd(t, t->enc_a[0], t->enc_b[0], t->E[0].c, H(0), W(0), t->E[0].za, t->E[0].t, t->E[0].go, t->E[0].gc, st);
  cbs_bwd(t, t->enc_stem, kS1, t->media_b, H(0), W(0), t->E[0].z, t->E[0].gc, H(0), W(0), nullptr, st);
  return HS_OK;
}

int tfail(int code, const char* m) { return set_error(code, m); }

}  // namespace
}  // namespace hs

extern "C" {

HS_API size_t hs_train_param_count(const hs_train_desc_t* d) {
  if (!d || d->levels < 2 || d->levels > 8) return 0;
  hs_trainer t;
  t.d = *d;
  t.L = d->levels;
  hs::build_layout(&t);
  return t.nparam;
}

HS_API int hs_trainer_create(hs_trainer_t** out, const hs_train_desc_t* d, const float* params, void* stream) {
  using namespace hs;
  if (!out || !d || !params) return tfail(HS_ECONFIG, "null argument");
  const int L = d->levels;
  if (L < 2 || L > 8) return tfail(HS_ECONFIG, "levels must be in [2, 8]");
  for (int l = 0; l < L; ++l)
    if (d->channels[l] < 1 || d->channels[l] > 256 || (256 % d->channels[l]))
      return tfail(HS_ECONFIG, "channel counts must be powers of two <= 256");
  if (d->channels[L - 1] % 2) return tfail(HS_ECONFIG, "coarsest channel count must be even");
  const int ix = d->nx - 1, iy = d->ny - 1, f = 1 << (L - 1);
  if (ix < 1 || iy < 1 || ix % f || iy % f) return tfail(HS_EDIMENSION, "grid not divisible by 2^(levels-1)");
  if (ix / f < 3 || iy / f < 3) return tfail(HS_EDIMENSION, "coarse size too small");
  if (d->batch < 1) return tfail(HS_ECONFIG, "batch must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  hs_trainer* t = new hs_trainer;
  t->d = *d;
  t->L = L;
  t->ix = ix;
  t->iy = iy;
  t->B = d->batch;
  t->hc = ix / f;
  t->wc = iy / f;
  t->cc = d->channels[L - 1] / 2;
  build_layout(t);
  bool ok = true;
  auto A = [&](size_t n) {
    float* p = dalloc<float>(t, n);
    ok = ok && p;
    return p;
  };
  t->P = A(t->nparam);
  t->M = A(t->nparam);
  t->V = A(t->nparam);
  // gradient arena: parameter gradients + every activation gradient (zeroed once per step)
  const int B = t->B;
  size_t gbytes = 0;
  std::vector<size_t*> gslots;
  auto level_n = [&](int l, int c) { return (size_t)B * (ix >> l) * (iy >> l) * c; };
  size_t maxlev = 0;
  for (int l = 0; l < L; ++l) maxlev = std::max(maxlev, level_n(l, d->channels[l]));
  // grads of parameters
  size_t off_G = gbytes;
  gbytes += ((t->nparam * 4 + 255) / 256) * 256;
  size_t off_l[8][6];
  for (int l = 0; l < L; ++l) {
    const size_t n = ((level_n(l, d->channels[l]) * 4 + 255) / 256) * 256;
    for (int k = 0; k < 6; ++k) {
      off_l[l][k] = gbytes;
      gbytes += n;
    }
  }
  size_t off_gimp = gbytes;
  gbytes += ((level_n(L - 1, d->channels[L - 1]) * 4 + 255) / 256) * 256;
  t->grad_arena = reinterpret_cast<char*>(dalloc<char>(t, gbytes));
  ok = ok && t->grad_arena;
  t->grad_arena_bytes = gbytes;
  if (ok) {
    t->G = reinterpret_cast<float*>(t->grad_arena + off_G);
    for (int l = 0; l < L; ++l) {
      t->E[l].gc = reinterpret_cast<float*>(t->grad_arena + off_l[l][0]);
      t->E[l].go = reinterpret_cast<float*>(t->grad_arena + off_l[l][1]);
      t->S[l].gc = reinterpret_cast<float*>(t->grad_arena + off_l[l][2]);
      t->S[l].go = reinterpret_cast<float*>(t->grad_arena + off_l[l][3]);
      // U[l + 1] lives at level l
      if (l + 1 < L) {
        t->U[l + 1].gc = reinterpret_cast<float*>(t->grad_arena + off_l[l][4]);
        t->U[l + 1].go = reinterpret_cast<float*>(t->grad_arena + off_l[l][5]);
      }
    }
    t->gimp = reinterpret_cast<float*>(t->grad_arena + off_gimp);
  }
  for (int l = 0; l < L; ++l) {
    const size_t n = level_n(l, d->channels[l]);
    t->E[l].z = A(n), t->E[l].c = A(n), t->E[l].za = A(n), t->E[l].t = A(n), t->E[l].o = A(n);
    t->S[l].z = A(n), t->S[l].c = A(n), t->S[l].za = A(n), t->S[l].t = A(n), t->S[l].o = A(n);
    if (l + 1 < L) t->U[l + 1].z = A(n), t->U[l + 1].c = A(n), t->U[l + 1].za = A(n), t->U[l + 1].t = A(n),
                   t->U[l + 1].o = A(n);
  }
  t->media_b = A((size_t)B * ix * iy * 2);
  t->r2 = A((size_t)B * ix * iy * 2);
  t->out = A((size_t)B * ix * iy * 2);
  t->gout = A((size_t)B * ix * iy * 2);
  t->imp = A(level_n(L - 1, d->channels[L - 1]));
  t->scr_t = A(maxlev);
  t->scr_z = A(maxlev);
  t->s0 = A(256);
  t->s1 = A(256);
  t->zero_bias = A(256);
  // tensor-core weight layouts, re-packed from the parameters at the start of every step
  std::vector<Repack> tab;
  auto pack = [&](LayerP& p) {
    if (!ok) return;
    const size_t n = (size_t)p.cin * p.cout * 9;
    p.wf = A(n);
    p.wd = A(n);
    tab.push_back({t->P + p.w, p.wf, p.cout, p.cin, p.kind == kT2 ? 1 : 0, 0});
    if (p.kind == kS1) tab.push_back({t->P + p.w, p.wd, p.cin, p.cout, 1, 1});
    else if (p.kind == kS2) tab.push_back({t->P + p.w, p.wd, p.cin, p.cout, 1, 0});
    else tab.push_back({t->P + p.w, p.wd, p.cin, p.cout, 0, 0});
  };
  pack(t->enc_stem), pack(t->sol_stem), pack(t->head);
  for (int l = 0; l < L; ++l) pack(t->enc_a[l]), pack(t->enc_b[l]), pack(t->sol_a[l]), pack(t->sol_b[l]);
  for (int l = 1; l < L; ++l) pack(t->enc_down[l]), pack(t->sol_down[l]), pack(t->up[l]), pack(t->ures_a[l]),
                              pack(t->ures_b[l]);
  t->n_repack = (int)tab.size();
  t->repack = dalloc<Repack>(t, tab.size());
  ok = ok && t->repack;
  if (ok) cudaMemcpy(t->repack, tab.data(), tab.size() * sizeof(Repack), cudaMemcpyHostToDevice);
  // batch statistics per BN layer
  auto stat = [&](LayerP& p) {
    if (!p.bn) return;
    p.st_mean = A(p.cout);
    p.st_inv = A(p.cout);
  };
  stat(t->enc_stem), stat(t->sol_stem);
  for (int l = 0; l < L; ++l) stat(t->enc_a[l]), stat(t->sol_a[l]);
  for (int l = 1; l < L; ++l) stat(t->enc_down[l]), stat(t->sol_down[l]), stat(t->up[l]), stat(t->ures_a[l]);
  t->chan_part_cap = 2LL * 4 * 148 * 256;
  t->chan_part = dalloc<double>(t, t->chan_part_cap);
  t->wg_part_cap = 8LL << 20;
  t->wg_part = A(t->wg_part_cap);
  t->loss_part = dalloc<double>(t, 2048);
  t->loss_dev = dalloc<double>(t, 1);
  t->model_dev = dalloc<int>(t, B);
  const long long per_b = (long long)t->cc * 4 * t->hc * t->wc;
  t->Xf = dalloc<cufftComplex>(t, B * per_b);
  t->Yb = dalloc<cufftComplex>(t, B * per_b);
  t->spec = dalloc<cufftComplex>(t, per_b);
  const int gh = 2 * t->hc, gw = 2 * t->wc, bh = 3 * gh, bw = 3 * gw;
  t->big1 = dalloc<double2>(t, (size_t)t->cc * bh * bw);
  t->big2 = dalloc<double2>(t, (size_t)t->cc * bh * bw);
  t->gG = dalloc<double2>(t, (size_t)per_b);
  ok = ok && t->chan_part && t->wg_part && t->loss_part && t->loss_dev && t->model_dev && t->Xf && t->Yb && t->spec &&
       t->big1 && t->big2 && t->gG;
  if (!ok) {
    delete t;
    return tfail(HS_ECUDA, "trainer allocation");
  }
  int nB[2] = {gh, gw}, n1[2] = {bh, bw};
  if (cufftPlanMany(&t->pB, 2, nB, nullptr, 1, gh * gw, nullptr, 1, gh * gw, CUFFT_C2C, B * t->cc) != CUFFT_SUCCESS ||
      cufftPlanMany(&t->p1, 2, n1, nullptr, 1, bh * bw, nullptr, 1, bh * bw, CUFFT_Z2Z, t->cc) != CUFFT_SUCCESS ||
      cufftPlanMany(&t->p2, 2, nB, nullptr, 1, gh * gw, nullptr, 1, gh * gw, CUFFT_Z2Z, t->cc) != CUFFT_SUCCESS) {
    delete t;
    return tfail(HS_ECUDA, "cufft plan");
  }
  t->plans = true;
  cufftSetStream(t->pB, st);
  cufftSetStream(t->p1, st);
  cufftSetStream(t->p2, st);
  cudaMemcpyAsync(t->P, params, t->nparam * sizeof(float), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(t->M, 0, t->nparam * sizeof(float), st);
  cudaMemsetAsync(t->V, 0, t->nparam * sizeof(float), st);
  cudaMemsetAsync(t->G, 0, t->nparam * sizeof(float), st);
  cudaMemsetAsync(t->zero_bias, 0, 256 * sizeof(float), st);
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    delete t;
    return tfail(HS_ECUDA, cudaGetErrorString(cudaGetLastError()));
  }
  *out = t;
  return HS_OK;
}

HS_API void hs_trainer_destroy(hs_trainer_t* t) { delete t; }

HS_API int hs_trainer_step(hs_trainer_t* t, const float* media, int n_models, const int* model_of, const void* r,
                           const void* e, const hs_adam_t* adam, double* loss, void* stream) {
  using namespace hs;
  if (!t || !media || !model_of || !r || !e) return tfail(HS_ECONFIG, "null argument");
  const int B = t->B;
  for (int b = 0; b < B; ++b)
    if (model_of[b] < 0 || model_of[b] >= n_models) return tfail(HS_EDIMENSION, "model_of out of range");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(t->model_dev, model_of, B * sizeof(int), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(t->grad_arena, 0, t->grad_arena_bytes, st);
  const long long np = (long long)B * t->ix * t->iy;
  k_tr_media<<<g1(np * 2), 256, 0, st>>>(media, t->model_dev, t->media_b, B, t->ix, t->iy);
  k_tr_r2<<<g1(np), 256, 0, st>>>(static_cast<const double2*>(r), t->r2, B, t->d.nx, t->d.ny, t->ix, t->iy);
  k_tr_repack<<<dim3(64, t->n_repack), 256, 0, st>>>(t->repack);
  prof::count(3);
  int rc = green_fwd(t, st);
  if (!rc) rc = forward(t, st);
  if (rc) return tfail(rc, "training forward");
  const double s = t->d.h * t->d.h / 64.0;
  const long long nn = (long long)B * t->d.nx * t->d.ny;
  const unsigned lb = (unsigned)std::min<long long>(2048, (nn + 255) / 256);
  k_tr_loss<<<lb, 256, 0, st>>>(t->out, static_cast<const double2*>(e), t->gout, B, t->d.nx, t->d.ny, t->ix, t->iy, s,
                                t->loss_part);
  k_tr_loss_fin<<<1, 32, 0, st>>>(t->loss_part, (int)lb, B, t->loss_dev);
  prof::count(2);
  rc = backward(t, st);
  if (rc) return tfail(rc, "training backward");
  if (adam) {
    t->t += 1;
    const float c1 = (float)(1.0 - std::pow((double)adam->beta1, t->t));
    const float c2 = (float)(1.0 - std::pow((double)adam->beta2, t->t));
    k_tr_adam<<<g1((long long)t->nparam), 256, 0, st>>>(t->P, t->G, t->M, t->V, (long long)t->nparam, adam->lr,
                                                        adam->beta1, adam->beta2, adam->eps, c1, c2);
    prof::count(1);
  }
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return tfail(HS_ECUDA, cudaGetErrorString(err));
  if (loss) {
    if (cudaMemcpyAsync(loss, t->loss_dev, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return tfail(HS_ECUDA, "loss readback");
    if (!std::isfinite(*loss)) return tfail(HS_ENONFINITE, "non-finite training loss");
  }
  return HS_OK;
}

// data-parallel training: copy the flat gradient vector to (to_trainer = 0) or from (1) a caller
// device buffer, so an all-reduce (NCCL) can run between the backward pass and hs_trainer_apply
HS_API int hs_trainer_grads(hs_trainer_t* t, void* dev, int to_trainer, void* stream) {
  if (!t || !dev) return hs::tfail(HS_ECONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const cudaError_t e = to_trainer ? cudaMemcpyAsync(t->G, dev, t->nparam * sizeof(float), cudaMemcpyDeviceToDevice, st)
                                   : cudaMemcpyAsync(dev, t->G, t->nparam * sizeof(float), cudaMemcpyDeviceToDevice, st);
  return e == cudaSuccess ? HS_OK : hs::tfail(HS_ECUDA, cudaGetErrorString(e));
}

// one Adam step on the current gradient vector (after hs_trainer_step with adam = NULL)
HS_API int hs_trainer_apply(hs_trainer_t* t, const hs_adam_t* adam, void* stream) {
  if (!t || !adam) return hs::tfail(HS_ECONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  t->t += 1;
  const float c1 = (float)(1.0 - std::pow((double)adam->beta1, t->t));
  const float c2 = (float)(1.0 - std::pow((double)adam->beta2, t->t));
  hs::k_tr_adam<<<hs::g1((long long)t->nparam), 256, 0, st>>>(t->P, t->G, t->M, t->V, (long long)t->nparam, adam->lr,
                                                              adam->beta1, adam->beta2, adam->eps, c1, c2);
  hs::prof::count(1);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HS_OK : hs::tfail(HS_ECUDA, cudaGetErrorString(e));
}

// which: 0 parameters (incl. running statistics), 1 gradients of the last step, 2 Adam m, 3 Adam v
HS_API int hs_trainer_read(const hs_trainer_t* t, int which, float* host, void* stream) {
  if (!t || !host || which < 0 || which > 3) return hs::tfail(HS_ECONFIG, "bad read request");
  const float* src = which == 0 ? t->P : which == 1 ? t->G : which == 2 ? t->M : t->V;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(host, src, t->nparam * sizeof(float), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return hs::tfail(HS_ECUDA, "trainer read");
  return HS_OK;
}

// which: 0 parameters, 2 Adam m, 3 Adam v (checkpoint restore); step counter set by `step`
HS_API int hs_trainer_write(hs_trainer_t* t, int which, const float* host, int step, void* stream) {
  if (!t || !host || which == 1 || which < 0 || which > 3) return hs::tfail(HS_ECONFIG, "bad write request");
  float* dst = which == 0 ? t->P : which == 2 ? t->M : t->V;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(dst, host, t->nparam * sizeof(float), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return hs::tfail(HS_ECUDA, "trainer write");
  if (step >= 0) t->t = step;
  return HS_OK;
}

}  // extern "C"
