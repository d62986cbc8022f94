// bt200 -- CP-ALS of an SM-sized tensor on a thread-block cluster (C1: 32^3,
// R = 8; decomp.py:344-410).  Included by cp.cu inside its anonymous
// namespace (it uses spd_inv_gj / pinv_block / small_block_sum).
//
// The one-CTA kernel (cp_small_kernel) re-reads X from L2 twice per sweep
// and runs on one SM.  Here a cluster of CS = 8 CTAs keeps X in distributed
// shared memory for the whole run: CTA c owns the mode-1 slab
// X[c Ic : (c+1) Ic, :, :] (C1: 32 KB).  Per sweep
//
//   mode 1  P_slab = X_slab x3 C on DMMA, M1 rows of the slab, the slab's
//           rows of A = M1 pinv(V) written into every CTA (DSMEM);
//   mode 2  partial M2 over the slab's i from P_slab, all-gathered;
//   mode 3  partial M3 = X_slab^T (A o B) on DMMA, all-gathered;
//
// one cluster barrier per mode; everything after a gather (sum of the CS
// partials in rank order, F = M pinv(V), Gram, norms, the fit) is computed
// by every CTA redundantly in the same order, so all CTAs hold identical
// factors and take identical decisions (stop, explicit fit) without further
// exchange.  Warp 0 of every CTA runs the pinv of the mode while warps
// 1..15 run its MTTKRP.  No atomics: bit-reproducible.

namespace cg = cooperative_groups;

constexpr int CL_CS = 8;   // CTAs per cluster (portable maximum)

__device__ long long g_cluster_clk[16];  // rank 0's phase clocks of sweep 1 (tools/prof_c1_cluster.py)

struct ClusterLayout {
  int64_t xs, ps, f[3], m, g, vp, gbuf, nrm, smf, red, fun, fuloc, gat[2], part, resb, total;
  int Ic, ldk, ldf;
};

__host__ __device__ inline ClusterLayout cluster_layout(int64_t I, int64_t J, int64_t K, int64_t R,
                                                        int NP) {
  ClusterLayout l{};
  int64_t o = 0;
  auto take = [&](int64_t n) {
    const int64_t at = o;
    o += (n + 1) / 2 * 2;
    return at;
  };
  l.Ic = static_cast<int>((I + CL_CS - 1) / CL_CS);
  const int64_t K4 = (K + 3) / 4 * 4;
  l.ldk = bt_ld(static_cast<int>(K4));
  l.ldf = NP + 4;
  const int64_t rows = (l.Ic * J + 7) / 8 * 8;
  const int64_t mx = I > J ? (I > K ? I : K) : (J > K ? J : K);
  l.xs = take(rows * l.ldk);
  l.ps = take(rows * NP);
  l.f[0] = take(I * l.ldf);
  l.f[1] = take(J * l.ldf);
  l.f[2] = take((K4 + 8) * l.ldf);
  l.m = take(mx * NP);
  l.g = take(3 * R * R);
  l.vp = take(R * R);
  l.gbuf = take(NP * NP);
  l.nrm = take(NP);
  l.smf = take(3 * NP * (NP + 1));
  l.red = take(64);
  l.fun = take(I * NP);                 // mode 1: rows written by their owners (remote stores)
  l.fuloc = take(mx * NP);              // modes 2, 3: F_un, local
  l.gat[0] = take(CL_CS * J * NP);      // mode 2 partials [rank][J][NP]
  l.gat[1] = take(CL_CS * K * NP);      // mode 3 partials [rank][K][NP]
  const int64_t mt = (K + 7) / 8;
  const int64_t ch = mt < 15 ? 15 / mt : 1;
  l.part = take(ch * mt * 8 * NP);      // mode-3 chunk partials inside the CTA
  l.resb = take(CL_CS);
  l.total = o;
  (void)R;
  return l;
}

template <int NP>
__global__ void __launch_bounds__(512)
    cp_cluster_kernel(const double* __restrict__ X, int I, int J, int K, int R,
                      double* __restrict__ ga, double* __restrict__ gb, double* __restrict__ gc,
                      double* __restrict__ glam, double x2, int max_iters, double tol, int fit_mode,
                      double* __restrict__ fit_hist, int* __restrict__ out_info) {
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const ClusterLayout L = cluster_layout(I, J, K, R, NP);
  const int LDK = L.ldk, LDF = L.ldf, Ic = L.Ic;
  double* xs = sm + L.xs;
  double* P = sm + L.ps;
  double* F[3] = {sm + L.f[0], sm + L.f[1], sm + L.f[2]};
  double* M = sm + L.m;
  double* G[3] = {sm + L.g, sm + L.g + R * R, sm + L.g + 2 * R * R};
  double* Vp = sm + L.vp;
  double* gbuf = sm + L.gbuf;
  double* nrm = sm + L.nrm;
  double* smf = sm + L.smf;
  double* red = sm + L.red;
  double* fun = sm + L.fun;
  double* fuloc = sm + L.fuloc;
  double* gat[2] = {sm + L.gat[0], sm + L.gat[1]};
  double* part = sm + L.part;
  double* resb = sm + L.resb;
  __shared__ int stop, pinv_ok;
  __shared__ double fit_s, explicit_s;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int rowsn[3] = {I, J, K};
  const int K4 = (K + 3) / 4 * 4;
  const int i0 = rank * Ic;
  const int ni = i0 < I ? (I - i0 < Ic ? I - i0 : Ic) : 0;   // slab rows (mode 1)
  const int srows = ni * J;                                  // (i, j) rows of the slab
  const int srows8 = (Ic * J + 7) / 8 * 8;

  // ---- load the slab of X (zero padded), the initial factors, their Grams
  for (int e = tid; e < srows8 * LDK; e += nt) {
    const int row = e / LDK, k = e - row * LDK;
    xs[e] = (row < srows && k < K) ? X[((int64_t)i0 * J + row) * K + k] : 0.0;
  }
  {
    const double* gsrc[3] = {ga, gb, gc};
    for (int m = 0; m < 3; ++m) {
      const int nrows = m == 2 ? K4 + 8 : rowsn[m];
      for (int e = tid; e < nrows * LDF; e += nt) {
        const int row = e / LDF, c = e - row * LDF;
        F[m][e] = (row < rowsn[m] && c < R) ? gsrc[m][row * R + c] : 0.0;
      }
    }
  }
  if (tid == 0) stop = 0;
  __syncthreads();
  for (int m = 0; m < 3; ++m)
    for (int e = tid; e < R * R; e += nt) {
      const int a = e / R, b = e % R;
      double s = 0.0;
      for (int r = 0; r < rowsn[m]; ++r) s = fma(F[m][r * LDF + a], F[m][r * LDF + b], s);
      G[m][e] = s;
    }
  __syncthreads();
  cluster.sync();   // every CTA is resident before the first remote store

  auto pinv_w0 = [&](int go0, int go1) {
    if (warp == 0) {
      const bool ok = spd_inv_gj<NP>(G[go0], G[go1], R, Vp);
      if (tid == 0) pinv_ok = ok ? 1 : 0;
    }
  };
  // after M (rows x NP, all rows) is complete in this CTA: F_un = M Vp, Gram,
  // norms, normalised factor k and Gram; last: inner = <F_un, M>, fit
  auto finish = [&](int k, int go0, int go1, bool gathered, bool last) {
    // gathered: F_un already in fun (mode 1, rows stored by their owners);
    // else F_un = M Vp into the local buffer (fun may already be receiving
    // the next sweep's mode-1 rows from faster peers)
    const int nr = rowsn[k];
    double* fu = gathered ? fun : fuloc;
    if (!gathered) {
      if (!pinv_ok) {
        pinv_block<NP>(G[go0], G[go1], R, Vp, smf);
        __syncthreads();
      }
      for (int e = tid; e < nr * NP; e += nt) {
        const int row = e / NP, c = e % NP;
        double s = 0.0;
        if (c < R)
          for (int q = 0; q < R; ++q) s = fma(M[row * NP + q], Vp[q * R + c], s);
        fu[e] = s;
      }
      __syncthreads();
    }
    for (int e = tid; e < R * R; e += nt) {
      const int a = e / R, b = e % R;
      double s = 0.0;
      for (int r = 0; r < nr; ++r) s = fma(fu[r * NP + a], fu[r * NP + b], s);
      gbuf[e] = s;
    }
    // last: <F_un, M> and ||Xhat||^2 = sum(G0 o G1 o F_un^T F_un) (the column
    // norms cancel against the normalised Gram) in one block reduction
    double s_in = 0.0, s_xh = 0.0;
    if (last)
      for (int e = tid; e < nr * NP; e += nt) s_in = fma(fu[e], M[e], s_in);
    __syncthreads();
    if (last) {
      for (int e = tid; e < R * R; e += nt) s_xh += G[0][e] * G[1][e] * gbuf[e];
      s_in = warp_sum(s_in);
      s_xh = warp_sum(s_xh);
      if (lane == 0) {
        red[warp] = s_in;
        red[16 + warp] = s_xh;
      }
    }
    for (int r = tid; r < NP; r += nt) {
      double v = r < R ? sqrt(gbuf[r * R + r]) : 1.0;
      if (v == 0.0) v = 1.0;
      nrm[r] = v;
    }
    __syncthreads();
    for (int e = tid; e < R * R; e += nt) G[k][e] = gbuf[e] / (nrm[e / R] * nrm[e % R]);
    for (int e = tid; e < nr * NP; e += nt) {
      const int row = e / NP, c = e % NP;
      F[k][row * LDF + c] = fu[e] / nrm[c];
    }
    if (last && tid == 0) {
      double inner = 0.0, xh2 = 0.0;
      for (int w = 0; w < 16; ++w) {
        inner += red[w];
        xh2 += red[16 + w];
      }
      const double res2 = fmax(x2 - 2.0 * inner + xh2, 0.0);
      const double relres = sqrt(res2 / x2);
      explicit_s = ((fit_mode == 1) || (fit_mode == 0 && relres < 1e-3)) ? 1.0 : 0.0;
      fit_s = 1.0 - relres;
    }
    __syncthreads();
  };
  // sum the CS gathered partials (rank order) into M
  auto sum_gather = [&](const double* gb_, int nr) {
    for (int e = tid; e < nr * NP; e += nt) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < CL_CS; ++c) s += gb_[c * nr * NP + e];
      M[e] = s;
    }
    __syncthreads();
  };

  double prev = -INFINITY;
  int conv = 0, it = 0;
  int ck = 0;
#define CL_CLK() do { if (it == 1 && rank == 0 && tid == 0) g_cluster_clk[ck] = clock64(); ++ck; } while (0)
  for (it = 0; it < max_iters; ++it) {
    ck = 0;
    CL_CLK();
    // ------------------------------------------------------------ mode 1
    pinv_w0(1, 2);
    if (warp >= 1) {
      // P_slab = X_slab x3 C: warp per 8-row tile, NP / 8 column tiles
      for (int m0 = (warp - 1) * 8; m0 < srows; m0 += 15 * 8) {
        double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
        const double* xr = xs + (m0 + gq) * LDK + tq;
        const double* cr = F[2] + tq * LDF + gq;
        for (int k0 = 0; k0 < K4; k0 += 4) {
          const double av = xr[k0];
          dmma884(c00, c01, av, cr[k0 * LDF]);
          if (NP > 8) dmma884(c10, c11, av, cr[k0 * LDF + 8]);
        }
        double* pr = P + (m0 + gq) * NP + 2 * tq;
        pr[0] = c00;
        pr[1] = c01;
        if (NP > 8) {
          pr[8] = c10;
          pr[9] = c11;
        }
      }
    }
    __syncthreads();
    CL_CLK();
    // M1 rows of the slab
    for (int e = tid; e < ni * NP; e += nt) {
      const int il = e / NP, r = e % NP;
      double s = 0.0;
      for (int j = 0; j < J; ++j) s = fma(P[(il * J + j) * NP + r], F[1][j * LDF + r], s);
      M[e] = s;
    }
    if (!pinv_ok) {
      __syncthreads();
      pinv_block<NP>(G[1], G[2], R, Vp, smf);
    }
    __syncthreads();
    // the slab's rows of F_un = M1 Vp, stored into every CTA's fun
    for (int e = tid; e < ni * NP; e += nt) {
      const int il = e / NP, c = e % NP;
      double s = 0.0;
      if (c < R)
        for (int q = 0; q < R; ++q) s = fma(M[il * NP + q], Vp[q * R + c], s);
      const int off = (i0 + il) * NP + c;
#pragma unroll
      for (int d = 0; d < CL_CS; ++d) cluster.map_shared_rank(fun, d)[off] = s;
    }
    CL_CLK();
    cluster.sync();
    CL_CLK();
    finish(0, 1, 2, true, false);
    CL_CLK();
    // ------------------------------------------------------------ mode 2
    pinv_w0(0, 2);
    if (warp >= 1) {
      for (int e = tid - 32; e < J * NP; e += nt - 32) {
        const int j = e / NP, r = e % NP;
        double s = 0.0;
        for (int il = 0; il < ni; ++il) s = fma(P[(il * J + j) * NP + r], F[0][(i0 + il) * LDF + r], s);
#pragma unroll
        for (int d = 0; d < CL_CS; ++d) cluster.map_shared_rank(gat[0], d)[rank * J * NP + e] = s;
      }
    }
    CL_CLK();
    cluster.sync();
    CL_CLK();
    sum_gather(gat[0], J);
    finish(1, 0, 2, false, false);
    CL_CLK();
    // ------------------------------------------------------------ mode 3
    pinv_w0(0, 1);
    {
      const int mtiles = (K + 7) / 8;
      const int chunks = mtiles < 15 ? 15 / mtiles : 1;
      const int clen = ((srows8 + chunks - 1) / chunks + 3) / 4 * 4;
      if (warp >= 1) {
        for (int item = warp - 1; item < mtiles * chunks; item += 15) {
          const int mt = item % mtiles, ch = item / mtiles;
          double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
          const int s0 = ch * clen, s1 = s0 + clen < srows8 ? s0 + clen : srows8;
          for (int r0 = s0; r0 < s1; r0 += 4) {
            const int row = r0 + tq;              // rows >= srows hold zeros in xs
            const int il = row / J, j = row - il * J;
            const int ia = i0 + il < I ? i0 + il : 0;
            const double av = xs[row * LDK + mt * 8 + gq];
            const double w0 = F[0][ia * LDF + gq] * F[1][j * LDF + gq];
            dmma884(c00, c01, av, w0);
            if (NP > 8) {
              const double w1 = F[0][ia * LDF + 8 + gq] * F[1][j * LDF + 8 + gq];
              dmma884(c10, c11, av, w1);
            }
          }
          double* pp = part + ((ch * mtiles + mt) * 8 + gq) * NP + 2 * tq;
          pp[0] = c00;
          pp[1] = c01;
          if (NP > 8) {
            pp[8] = c10;
            pp[9] = c11;
          }
        }
      }
      __syncthreads();
      for (int e = tid; e < K * NP; e += nt) {
        const int kk = e / NP, r = e % NP;
        double s = 0.0;
        for (int ch = 0; ch < chunks; ++ch) s += part[((ch * mtiles) * 8 + kk) * NP + r];
#pragma unroll
        for (int d = 0; d < CL_CS; ++d) cluster.map_shared_rank(gat[1], d)[rank * K * NP + e] = s;
      }
    }
    CL_CLK();
    cluster.sync();
    CL_CLK();
    sum_gather(gat[1], K);
    finish(2, 0, 1, false, true);
    CL_CLK();
    if (explicit_s != 0.0) {
      // ||X - [[A lam, B, C]]||^2 over the slab, gathered
      double loc = 0.0;
      for (int row = tid; row < srows; row += nt) {
        const int il = row / J, j = row - il * J;
        double wb[NP];
#pragma unroll
        for (int r = 0; r < NP; ++r) wb[r] = F[0][(i0 + il) * LDF + r] * nrm[r] * F[1][j * LDF + r];
        for (int kk = 0; kk < K; ++kk) {
          double xh = 0.0;
#pragma unroll
          for (int r = 0; r < NP; ++r) xh = fma(wb[r], F[2][kk * LDF + r], xh);
          const double d = xs[row * LDK + kk] - xh;
          loc = fma(d, d, loc);
        }
      }
      const double res_slab = small_block_sum(loc, red);
      if (tid < CL_CS) cluster.map_shared_rank(resb, tid)[rank] = res_slab;
      cluster.sync();
      if (tid == 0) {
        double res2 = 0.0;
        for (int c = 0; c < CL_CS; ++c) res2 += resb[c];
        fit_s = 1.0 - sqrt(res2) / sqrt(x2);
      }
      __syncthreads();
    }
    if (tid == 0) {
      const double fit = fit_s;
      if (rank == 0) fit_hist[it] = fit;
      if (tol > 0.0 && fabs(fit - prev) < tol) stop = 1;
      prev = fit;
    }
    __syncthreads();
    if (stop) {
      conv = 1;
      ++it;
      break;
    }
  }
#undef CL_CLK
  if (it > max_iters) it = max_iters;
  cluster.sync();   // no CTA exits while a peer may still store into it
  if (rank == 0) {
    for (int e = tid; e < I * R; e += nt) ga[e] = F[0][(e / R) * LDF + e % R] * nrm[e % R];
    for (int e = tid; e < J * R; e += nt) gb[e] = F[1][(e / R) * LDF + e % R];
    for (int e = tid; e < K * R; e += nt) gc[e] = F[2][(e / R) * LDF + e % R];
    for (int r = tid; r < R; r += nt) glam[r] = nrm[r];
    if (tid == 0) {
      out_info[0] = it;
      out_info[1] = conv;
    }
  }
}
