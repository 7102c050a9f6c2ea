// tiny.cu — the whole of Algorithm 1 in ONE warp for tiny QPs (n, m <= 64; C1).
//
// At n = 50 every IPM iteration of the multi-kernel path is ~16 launches and a host round trip
// around a ~1 us-per-iteration PCG: launch latency, not arithmetic, is the QP time (P:325 makes
// the same observation on the A100).  Here one 32-thread CTA keeps H, A (dense), the assembled K
// and every iterate vector in shared memory and runs, after the start point (ipmops.cu, R5/R15):
//   residuals (eq:perturbed_KKT, R1) -> Sigma_b, Sigma_c, Jacobi
//   -> condensed rhs (eq:2x2_reduced + Schur complement) -> PCG on K = H + A^T Sigma_c A + Sigma_b
//   (the one-warp loop of pcg.cu with its true-residual restarts) -> recovery and
//   fraction-to-boundary step lengths -> update -> residuals -> mu control (Alg. 1
//   lines 10-15), per-iteration trace records, the final report at the final mu.
// The formulas, their association where it matters (K, the recovery, the update) and every
// stopping rule are those of the multi-kernel path (ipmops.cu, pcg.cu, ipm_api.cu solve_impl);
// sums over a vector use a warp shuffle tree instead of a block tree, so results agree to
// rounding, not bitwise.  Predictor-corrector, PCG warm starts, the augmented system, compact
// Hessians and sharding stay on the multi-kernel path.
#include "ipm.h"
#include "common.cuh"
#include "kernels.h"
#include "state.h"

namespace ipm {

namespace {
__device__ __forceinline__ bool has(double b) { return fabs(b) < INFINITY; }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
constexpr int kT = kWarpMaxN;          // max n and m
constexpr int kLd = kT + 1;            // odd smem row stride: conflict-free row and column walks
constexpr int kNV = 25, kMV = 21;      // n- and m-space vectors in shared memory
}  // namespace

// sum_k u[k * su] v[k * sv], k < len, four FMA chains combined in a fixed order (latency-bound
// walks over shared memory otherwise dominate the non-PCG part of an IPM iteration)
__device__ __forceinline__ double dot4(const double *u, int su, const double *v, int sv, int len) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int k = 0;
    for (; k + 3 < len; k += 4) {
        a0 = fma(u[k * su], v[k * sv], a0);
        a1 = fma(u[(k + 1) * su], v[(k + 1) * sv], a1);
        a2 = fma(u[(k + 2) * su], v[(k + 2) * sv], a2);
        a3 = fma(u[(k + 3) * su], v[(k + 3) * sv], a3);
    }
    for (; k < len; ++k) a0 = fma(u[k * su], v[k * sv], a0);
    return (a0 + a1) + (a2 + a3);
}

size_t tiny_smem_bytes() { return 8 * ((size_t)3 * kT * kLd + (size_t)(kNV + kMV) * kT); }

bool tiny_eligible(int n, int m) { return n >= 1 && n <= kT && m >= 0 && m <= kT; }

__global__ void __launch_bounds__(32, 1) k_ipm_tiny(TinyArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int l = threadIdx.x;
    const int n = a.n, m = a.m;
    double *sH = sm, *sK = sH + kT * kLd, *sA = sK + kT * kLd, *v = sA + kT * kLd;
    // n-space
    double *x = v, *slx = x + kT, *sux = slx + kT, *llx = sux + kT, *lux = llx + kT, *xl = lux + kT, *xu = xl + kT,
           *g = xu + kT, *rH = g + kT, *rlx = rH + kT, *rux = rlx + kT, *rclx = rux + kT, *rcux = rclx + kT,
           *sigb = rcux + kT, *minv = sigb + kT, *rhs = minv + kT, *dx = rhs + kT, *sp = dx + kT, *dslx = sp + kT,
           *dsux = dslx + kT, *dllx = dsux + kT, *dlux = dllx + kT, *hx = dlux + kT, *rv = hx + kT, *zv = rv + kT;
    // m-space
    double *w0 = v + kNV * kT;
    double *lo = w0, *hi = lo + kT, *slA = hi + kT, *suA = slA + kT, *llA = suA + kT, *luA = llA + kT, *Ax = luA + kT,
           *rlA = Ax + kT, *ruA = rlA + kT, *lamd = ruA + kT, *sigc = lamd + kT, *rclA = sigc + kT, *rcuA = rclA + kT,
           *r2l = rcuA + kT, *r2u = r2l + kT, *wv = r2u + kT, *Adx = wv + kT, *dslA = Adx + kT, *dsuA = dslA + kT,
           *dllA = dsuA + kT, *dluA = dllA + kT;

    // ---- stage the problem and the start point
    for (int i = 0; i < n; ++i)
        for (int j = l; j < n; j += 32) sH[i * kLd + j] = a.H[(int64_t)i * a.ldh + j];
    for (int i = 0; i < m; ++i) {
        for (int j = l; j < n; j += 32) sA[i * kLd + j] = 0.0;
        __syncwarp();
        for (int64_t k = a.Arp[i] + l; k < a.Arp[i + 1]; k += 32) sA[i * kLd + a.Acol[k]] = a.Aval[k];
    }
    for (int j = l; j < n; j += 32) {
        x[j] = a.x[j]; slx[j] = a.s_lx[j]; sux[j] = a.s_ux[j]; llx[j] = a.lam_lx[j]; lux[j] = a.lam_ux[j];
        xl[j] = a.xl[j]; xu[j] = a.xu[j]; g[j] = a.g[j];
    }
    for (int i = l; i < m; i += 32) {
        lo[i] = a.l[i]; hi[i] = a.u[i]; slA[i] = a.s_lA[i]; suA[i] = a.s_uA[i]; llA[i] = a.lam_lA[i]; luA[i] = a.lam_uA[i];
    }
    __syncwarp();

    double rh_max = 0.0, prim_max = 0.0, comp_max = 0.0, ls_max = 0.0, obj = 0.0;
    int nonfinite = 0;
    // ---- residuals at mu (ipmops.cu k_resid_m / k_resid_n)
    auto residuals = [&](double mu) {
        for (int i = l; i < m; i += 32) Ax[i] = dot4(sA + i * kLd, 1, x, 1, n);
        double prim = 0.0, comp = 0.0, lsm = 0.0, rhm = 0.0, ob = 0.0;
        int bad = 0;
        for (int i = l; i < m; i += 32) {
            const double ax = Ax[i];
            double rl = 0.0, ru = 0.0;
            if (has(lo[i])) {
                rl = ax - slA[i] - lo[i];
                const double ls = llA[i] * slA[i];
                prim = fmax(prim, fabs(rl));
                comp = fmax(comp, fabs(ls - mu));
                lsm = fmax(lsm, ls);
                bad |= !finite_d(rl) | !finite_d(ls);
            }
            if (has(hi[i])) {
                ru = hi[i] - ax - suA[i];
                const double ls = luA[i] * suA[i];
                prim = fmax(prim, fabs(ru));
                comp = fmax(comp, fabs(ls - mu));
                lsm = fmax(lsm, ls);
                bad |= !finite_d(ru) | !finite_d(ls);
            }
            rlA[i] = rl;
            ruA[i] = ru;
            lamd[i] = llA[i] - luA[i];
        }
        __syncwarp();
        for (int j = l; j < n; j += 32) {
            const double hs = dot4(sH + j * kLd, 1, x, 1, n), at = dot4(sA + j, kLd, lamd, 1, m);
            const double xj = x[j];
            hx[j] = hs;
            const double r = hs + g[j] - at - llx[j] + lux[j];
            rH[j] = r;
            rhm = fmax(rhm, fabs(r));
            bad |= !finite_d(r);
            ob = fma(0.5 * xj, hs, ob);
            ob = fma(g[j], xj, ob);
            double rl = 0.0, ru = 0.0;
            if (has(xl[j])) {
                rl = xj - slx[j] - xl[j];
                const double ls = llx[j] * slx[j];
                prim = fmax(prim, fabs(rl));
                comp = fmax(comp, fabs(ls - mu));
                lsm = fmax(lsm, ls);
                bad |= !finite_d(rl) | !finite_d(ls);
            }
            if (has(xu[j])) {
                ru = xu[j] - xj - sux[j];
                const double ls = lux[j] * sux[j];
                prim = fmax(prim, fabs(ru));
                comp = fmax(comp, fabs(ls - mu));
                lsm = fmax(lsm, ls);
                bad |= !finite_d(ru) | !finite_d(ls);
            }
            rlx[j] = rl;
            rux[j] = ru;
        }
        rh_max = warp_max(rhm);
        prim_max = warp_max(prim);
        comp_max = warp_max(comp);
        ls_max = warp_max(lsm);
        obj = warp_sum(ob);
        if (__any_sync(0xffffffffu, bad) || !finite_d(obj)) nonfinite = 1;
        __syncwarp();
    };

    // ---- one Newton direction into dx (Alg. 1 lines 2-3): Sigma's, rhs, PCG on the assembled K
    int64_t pcg_it = 0;
    int pcg_restarts = 0, pcg_stalled = 0, pcg_breakdown = 0;
    double pcg_relres = 0.0;
    auto direction = [&](double mu, double rtol) {
        for (int i = l; i < m; i += 32) {
            double s = 0.0;
            if (has(lo[i])) s += llA[i] / slA[i];
            if (has(hi[i])) s += luA[i] / suA[i];
            sigc[i] = s;
        }
        __syncwarp();
        for (int j = l; j < n; j += 32) {
            double s0 = 0.0, s1 = 0.0;
            int i = 0;
            for (; i + 1 < m; i += 2) {
                const double a0 = sA[i * kLd + j], a1 = sA[(i + 1) * kLd + j];
                s0 = fma(a0 * a0, sigc[i], s0);
                s1 = fma(a1 * a1, sigc[i + 1], s1);
            }
            if (i < m) s0 = fma(sA[i * kLd + j] * sA[i * kLd + j], sigc[i], s0);
            const double s = s0 + s1;
            double sb = 0.0;
            if (has(xl[j])) sb += llx[j] / slx[j];
            if (has(xu[j])) sb += lux[j] / sux[j];
            sigb[j] = sb;
            minv[j] = 1.0 / (sH[j * kLd + j] + sb + s);
        }
        // condensed rhs, mode 0: r_c = lam s - mu
        for (int i = l; i < m; i += 32) {
            double wi = 0.0, ra = 0.0, rb = 0.0, ca = 0.0, cb = 0.0;
            if (has(lo[i])) {
                const double lam = llA[i], s = slA[i];
                ca = lam * s - mu;
                ra = -rlA[i] - ca / lam;
                wi += ra / (s / lam);
            }
            if (has(hi[i])) {
                const double lam = luA[i], s = suA[i];
                cb = lam * s - mu;
                rb = -ruA[i] - cb / lam;
                wi -= rb / (s / lam);
            }
            rclA[i] = ca;
            rcuA[i] = cb;
            r2l[i] = ra;
            r2u[i] = rb;
            wv[i] = wi;
        }
        __syncwarp();
        for (int j = l; j < n; j += 32) {
            const double at = dot4(sA + j, kLd, wv, 1, m);
            double r1 = -rH[j], ca = 0.0, cb = 0.0;
            if (has(xl[j])) {
                ca = llx[j] * slx[j] - mu;
                r1 -= fma(llx[j], rlx[j], ca) / slx[j];
            }
            if (has(xu[j])) {
                cb = lux[j] * sux[j] - mu;
                r1 += fma(lux[j], rux[j], cb) / sux[j];
            }
            rclx[j] = ca;
            rcux[j] = cb;
            rhs[j] = fma(1.0, at, r1);
        }
        // K = (H + sum_r sigma_r (A_rj A_rk)) + delta_jk sigma_b,j over the rows r with A_rj != 0 in
        // ascending r — k_form_K's terms and association, so the same bits.  Lane l builds columns
        // k = l, l + 32 for every j (the nonzero test on A_rj is warp-uniform: no divergence) and
        // stores K_jk at sK[k * kLd + j], the layout the PCG walks lane-consecutively.
        for (int j = 0; j < n; ++j) {
            double acc0 = 0.0, acc1 = 0.0;
            for (int r = 0; r < m; ++r) {
                const double arj = sA[r * kLd + j];
                if (arj == 0.0) continue;
                const double sr = sigc[r];
                acc0 = fma(sr, arj * sA[r * kLd + l], acc0);
                acc1 = fma(sr, arj * sA[r * kLd + l + 32], acc1);
            }
            if (l < n) sK[l * kLd + j] = (sH[j * kLd + l] + acc0) + (j == l ? sigb[j] : 0.0);
            if (l + 32 < n) sK[(l + 32) * kLd + j] = (sH[j * kLd + l + 32] + acc1) + (j == l + 32 ? sigb[j] : 0.0);
        }
        __syncwarp();
        // PCG from x0 = 0 (k_pcg_init), stopping rule S:225, restarts on the true residual — the
        // register-resident loop of k_pcg_warp: lane l owns rows l and l + 32, u broadcast from sp
        const int i0 = l, i1 = l + 32;
        const bool h0 = i0 < n, h1 = i1 < n;
        auto kmul = [&](const double *u, double &o0, double &o1) {   // (K u) rows i0, i1 (k_pcg_warp's)
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
            const int n4 = n & ~3;
            int k = 0;
#pragma unroll 4
            for (; k < n4; k += 4) {
                const double2 ua = *reinterpret_cast<const double2 *>(u + k);
                const double2 ub = *reinterpret_cast<const double2 *>(u + k + 2);
                const double *kr = sK + k * kLd;
                a0 = fma(kr[i0], ua.x, a0);
                c0 = fma(kr[i1], ua.x, c0);
                a1 = fma(kr[kLd + i0], ua.y, a1);
                c1 = fma(kr[kLd + i1], ua.y, c1);
                a2 = fma(kr[2 * kLd + i0], ub.x, a2);
                c2 = fma(kr[2 * kLd + i1], ub.x, c2);
                a3 = fma(kr[3 * kLd + i0], ub.y, a3);
                c3 = fma(kr[3 * kLd + i1], ub.y, c3);
            }
            for (; k < n; ++k) {
                a0 = fma(sK[k * kLd + i0], u[k], a0);
                c0 = fma(sK[k * kLd + i1], u[k], c0);
            }
            o0 = h0 ? (a0 + a1) + (a2 + a3) : 0.0;
            o1 = h1 ? (c0 + c1) + (c2 + c3) : 0.0;
        };
        const double b0 = h0 ? rhs[i0] : 0.0, b1 = h1 ? rhs[i1] : 0.0;
        const double m0 = h0 ? minv[i0] : 0.0, m1 = h1 ? minv[i1] : 0.0;
        double x0 = 0.0, x1 = 0.0, r0 = b0, r1 = b1, z0 = m0 * b0, z1 = m1 * b1, p0 = 0.0, p1 = 0.0;
        double rho = warp_sum(fma(r1, z1, r0 * z0)), rr = warp_sum(fma(r1, r1, r0 * r0)), rho_old = rho;
        const double rhs2 = rr;
        const double tol2 = fmax(rtol * rtol * rr, a.atol * a.atol);
        int64_t it = 0, it_rs = 0;
        const int64_t maxit = a.pcg_maxit > 0 ? a.pcg_maxit : 10 * (int64_t)n;
        int done = (rr <= tol2) ? 1 : 0, breakdown = (!finite_d(rr) || !finite_d(rho)) ? 1 : 0, stalled = 0, rs = 0;
        double res2 = 0.0;
        __syncwarp();
        for (int round = 0; !breakdown; ++round) {
            while (!done) {
                const bool first = (it_rs == 0);
                const double beta = first ? 0.0 : rho / rho_old;
                p0 = first ? z0 : fma(beta, p0, z0);
                p1 = first ? z1 : fma(beta, p1, z1);
                sp[i0] = p0;                     // 0 beyond n
                sp[i1] = p1;
                __syncwarp();
                double y0, y1;
                kmul(sp, y0, y1);
                const double pkp = warp_sum(fma(p0, y0, p1 * y1));
                if (!(pkp > 0.0) || !finite_d(pkp)) {
                    breakdown = 1;
                    break;
                }
                const double alpha = rho / pkp;
                x0 = fma(alpha, p0, x0);
                x1 = fma(alpha, p1, x1);
                r0 = fma(-alpha, y0, r0);
                r1 = fma(-alpha, y1, r1);
                z0 = m0 * r0;
                z1 = m1 * r1;
                double rz2 = fma(r1, z1, r0 * z0), rr2 = fma(r1, r1, r0 * r0);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    rz2 += __shfl_xor_sync(0xffffffffu, rz2, o);
                    rr2 += __shfl_xor_sync(0xffffffffu, rr2, o);
                }
                rho_old = rho;
                rho = rz2;
                rr = rr2;
                ++it;
                ++it_rs;
                if (!finite_d(rr) || !finite_d(rho)) {
                    breakdown = 1;
                    break;
                }
                done = (rr <= tol2 || it >= maxit) ? 1 : 0;
                __syncwarp();                    // sp reads done before the next overwrite
            }
            if (breakdown) break;
            // true residual with the same K
            __syncwarp();
            sp[i0] = x0;
            sp[i1] = x1;
            __syncwarp();
            double k0, k1;
            kmul(sp, k0, k1);
            const double t0 = h0 ? b0 - k0 : 0.0, t1 = h1 ? b1 - k1 : 0.0;
            res2 = warp_sum(fma(t1, t1, t0 * t0));
            if (!finite_d(res2) || res2 <= tol2) break;
            if (it >= maxit || round >= 8) {
                stalled = 1;
                break;
            }
            ++rs;
            r0 = t0;
            r1 = t1;
            z0 = m0 * r0;
            z1 = m1 * r1;
            rho = rho_old = warp_sum(fma(r1, z1, r0 * z0));
            rr = warp_sum(fma(r1, r1, r0 * r0));
            it_rs = 0;
            done = (rr <= tol2 || it >= maxit) ? 1 : 0;
            __syncwarp();
        }
        __syncwarp();
        if (h0) dx[i0] = x0;
        if (h1) dx[i1] = x1;
        pcg_it = it;
        pcg_restarts = rs;
        pcg_stalled = stalled;
        pcg_breakdown = breakdown;
        pcg_relres = rhs2 > 0 ? sqrt(res2 / rhs2) : 0.0;
        if (!breakdown && !finite_d(res2)) nonfinite = 2;   // non-finite PCG residual
        __syncwarp();
    };

    // ---- recovery + fraction to the boundary (ipmops.cu k_recover_m / k_recover_n) and update
    double alpha_x = 0.0, alpha_l = 0.0;
    auto step = [&](double tau) {
        for (int i = l; i < m; i += 32) Adx[i] = dot4(sA + i * kLd, 1, dx, 1, n);
        __syncwarp();
        double mx = INFINITY, ml = INFINITY;
        int bad = 0;
        auto rmin = [](double val, double dv, double &mn) {
            if (dv < 0.0) mn = fmin(mn, -val / dv);
        };
        for (int i = l; i < m; i += 32) {
            const double ad = Adx[i];
            double dsl = 0.0, dll = 0.0, dsu = 0.0, dlu = 0.0;
            if (has(lo[i])) {
                dsl = ad + rlA[i];
                dll = (r2l[i] - ad) / (slA[i] / llA[i]);
                rmin(slA[i], dsl, mx);
                rmin(llA[i], dll, ml);
                bad |= !finite_d(dsl) | !finite_d(dll);
            }
            if (has(hi[i])) {
                dsu = -ad + ruA[i];
                dlu = (r2u[i] + ad) / (suA[i] / luA[i]);
                rmin(suA[i], dsu, mx);
                rmin(luA[i], dlu, ml);
                bad |= !finite_d(dsu) | !finite_d(dlu);
            }
            dslA[i] = dsl; dsuA[i] = dsu; dllA[i] = dll; dluA[i] = dlu;
        }
        for (int j = l; j < n; j += 32) {
            const double d = dx[j];
            double dsl = 0.0, dll = 0.0, dsu = 0.0, dlu = 0.0;
            bad |= !finite_d(d);
            if (has(xl[j])) {
                dsl = d + rlx[j];
                dll = -fma(llx[j], dsl, rclx[j]) / slx[j];
                rmin(slx[j], dsl, mx);
                rmin(llx[j], dll, ml);
                bad |= !finite_d(dsl) | !finite_d(dll);
            }
            if (has(xu[j])) {
                dsu = -d + rux[j];
                dlu = -fma(lux[j], dsu, rcux[j]) / sux[j];
                rmin(sux[j], dsu, mx);
                rmin(lux[j], dlu, ml);
                bad |= !finite_d(dsu) | !finite_d(dlu);
            }
            dslx[j] = dsl; dsux[j] = dsu; dllx[j] = dll; dlux[j] = dlu;
        }
        if (__any_sync(0xffffffffu, bad)) nonfinite = 1;
        alpha_x = fmin(1.0, tau * warp_min(mx));
        alpha_l = fmin(1.0, tau * warp_min(ml));
        __syncwarp();
        for (int i = l; i < m; i += 32) {
            slA[i] = fma(alpha_x, dslA[i], slA[i]);
            suA[i] = fma(alpha_x, dsuA[i], suA[i]);
            llA[i] = fma(alpha_l, dllA[i], llA[i]);
            luA[i] = fma(alpha_l, dluA[i], luA[i]);
        }
        for (int j = l; j < n; j += 32) {
            x[j] = fma(alpha_x, dx[j], x[j]);
            slx[j] = fma(alpha_x, dslx[j], slx[j]);
            sux[j] = fma(alpha_x, dsux[j], sux[j]);
            llx[j] = fma(alpha_l, dllx[j], llx[j]);
            lux[j] = fma(alpha_l, dlux[j], lux[j]);
        }
        __syncwarp();
    };

    // ---- Algorithm 1 (ipm_api.cu solve_impl, non-Mehrotra branch)
    double mu = a.mu0;
    residuals(mu);
    int status = IPM_NOT_CONVERGED, k = 0;
    int64_t pcg_total = 0;
    int pcg_max = 0, stalls = 0, restarts = 0;
    unsigned long long t_pcg = 0;
    int ntrace = 0;
    if (nonfinite) {
        status = IPM_ERR_NONFINITE;
    } else {
        for (k = 1; k <= a.max_ipm; ++k) {
            const double rtol = a.schedule == 1 ? fmax(1e-10, fmin(1e-2, 0.1 * mu))
                                                : fmax(a.rtol_floor, fmin(a.rtol_max, a.rtol_fac * mu));
            const unsigned long long t0 = gtimer();
            direction(mu, rtol);
            t_pcg += gtimer() - t0;
            pcg_total += pcg_it;
            pcg_max = max(pcg_max, (int)pcg_it);
            stalls += pcg_stalled;
            restarts += pcg_restarts;
            if (pcg_breakdown) { status = IPM_ERR_PCG_BREAKDOWN; break; }
            if (nonfinite == 2) { status = IPM_ERR_NONFINITE; break; }
            step(a.tau);
            residuals(mu);
            const double nrm = fmax(rh_max, fmax(prim_max, comp_max));
            if (a.trace && l == 0) {
                ipm_trace_rec r;
                r.it = k;
                r.pcg_iters = (int32_t)pcg_it;
                r.mu = mu;
                r.kkt_inf = nrm;
                r.alpha_x = alpha_x;
                r.alpha_lam = alpha_l;
                r.pcg_relres = pcg_relres;
                r.obj = obj;
                reinterpret_cast<ipm_trace_rec *>(a.trace_buf)[k - 1] = r;
            }
            ntrace = k;
            if (nonfinite) { status = IPM_ERR_NONFINITE; break; }
            if (nrm < mu) {
                if (mu <= a.mu_tol) { status = IPM_OK; break; }
                mu = mu / a.mu_div;
            }
        }
    }
    if (status == IPM_OK || status == IPM_NOT_CONVERGED || status == IPM_ERR_NONFINITE) residuals(mu);   // report
    // ---- write back the iterate, the last direction and the scalars
    for (int j = l; j < n; j += 32) {
        a.x[j] = x[j]; a.s_lx[j] = slx[j]; a.s_ux[j] = sux[j]; a.lam_lx[j] = llx[j]; a.lam_ux[j] = lux[j];
        a.dx[j] = dx[j]; a.Hx[j] = hx[j];
    }
    for (int i = l; i < m; i += 32) {
        a.s_lA[i] = slA[i]; a.s_uA[i] = suA[i]; a.lam_lA[i] = llA[i]; a.lam_uA[i] = luA[i]; a.Ax[i] = Ax[i];
    }
    if (l == 0) {
        Scalars *sc = a.sc;
        sc->rH_max = rh_max;
        sc->prim_max = prim_max;
        sc->comp_max = comp_max;
        sc->ls_max = ls_max;
        sc->obj = obj;
        sc->alpha_x = alpha_x;
        sc->alpha_l = alpha_l;
        sc->nonfinite = nonfinite ? 1 : 0;
        TinyOut *o = a.out;
        o->status = status;
        o->ipm_iters = min(k, a.max_ipm);
        o->pcg_total = pcg_total;
        o->pcg_max = pcg_max;
        o->stalls = stalls;
        o->restarts = restarts;
        o->mu = mu;
        o->t_pcg_ns = t_pcg;
        o->pcg_it_last = pcg_it;
        o->ntrace = ntrace;
    }
}

void launch_ipm_tiny(const TinyArgs &a, cudaStream_t st) {
    k_ipm_tiny<<<1, 32, tiny_smem_bytes(), st>>>(a);
}

cudaError_t configure_tiny_attrs() {
    return cudaFuncSetAttribute(k_ipm_tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tiny_smem_bytes());
}

void preload_tiny() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, reinterpret_cast<const void *>(k_ipm_tiny));
}

}  // namespace ipm
