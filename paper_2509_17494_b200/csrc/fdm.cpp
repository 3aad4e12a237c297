// fdm.cpp -- fast diagonalisation of separable subdomain operators (host setup).
//
// A subdomain class whose Omega cells share one (k, eps) and whose sides are
// absorbing or Neumann has the exact tensor form
//   A_s^(Omega) = Kx (x) My + Mx (x) Ky,
//   Kx = Sx - i k h Ex,  Ky = Sy - i k h Ey - m My,  m = (k^2 (1 + i alpha_s) + i eps) h^2,
// (Ex, Ey: the absorbing end points; S, M: the 1-D hierarchical stiffness and
// mass assembled over the Omega cells). With the generalised eigenpairs
// K V = M V Lambda, V^T M V = I in each direction,
//   A^-1 = (Vx (x) Vy) diag(1 / (lx_i + ly_j)) (Vx (x) Vy)^T,
// so the U rows of A^-1 g cost four small dense products instead of one
// |U| x |Omega| product. The factors are validated against the dense
// restricted inverse of the same class before use.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>

#include "setup.hpp"
#include "kernels.hpp"

namespace htg {

namespace {

using Mat = std::vector<cplx>;  // row-major n x n

// Eigen-decomposition of a general complex matrix: Householder Hessenberg
// reduction, shifted QR (Wilkinson shifts, deflation) to the complex Schur
// form, eigenvectors of the triangular factor by back substitution.
bool complex_eig(int n, Mat A, std::vector<cplx>& lam, Mat& X) {
    auto at = [n](Mat& M, int i, int j) -> cplx& { return M[size_t(i) * n + j]; };
    Mat Q(size_t(n) * n, cplx(0.0));
    for (int i = 0; i < n; ++i) at(Q, i, i) = 1.0;
    // Hessenberg reduction
    for (int k = 0; k < n - 2; ++k) {
        double alpha2 = 0.0;
        for (int i = k + 1; i < n; ++i) alpha2 += std::norm(at(A, i, k));
        const double alpha = std::sqrt(alpha2);
        if (alpha == 0.0) continue;
        std::vector<cplx> v(n, cplx(0.0));
        const cplx x0 = at(A, k + 1, k);
        const cplx ph = std::abs(x0) > 0 ? x0 / std::abs(x0) : cplx(1.0);
        for (int i = k + 1; i < n; ++i) v[i] = at(A, i, k);
        v[k + 1] += ph * alpha;
        double vn = 0.0;
        for (int i = k + 1; i < n; ++i) vn += std::norm(v[i]);
        if (vn == 0.0) continue;
        // A = H A H, H = I - 2 v v^H / vn ; Q = Q H
        for (int j = 0; j < n; ++j) {
            cplx d = 0.0;
            for (int i = k + 1; i < n; ++i) d += std::conj(v[i]) * at(A, i, j);
            d *= 2.0 / vn;
            for (int i = k + 1; i < n; ++i) at(A, i, j) -= d * v[i];
        }
        for (int i = 0; i < n; ++i) {
            cplx d = 0.0;
            for (int j = k + 1; j < n; ++j) d += at(A, i, j) * v[j];
            d *= 2.0 / vn;
            for (int j = k + 1; j < n; ++j) at(A, i, j) -= d * std::conj(v[j]);
        }
        for (int i = 0; i < n; ++i) {
            cplx d = 0.0;
            for (int j = k + 1; j < n; ++j) d += at(Q, i, j) * v[j];
            d *= 2.0 / vn;
            for (int j = k + 1; j < n; ++j) at(Q, i, j) -= d * std::conj(v[j]);
        }
    }
    // shifted QR on the Hessenberg matrix with Givens rotations
    int hi = n - 1, iter = 0;
    while (hi > 0) {
        if (++iter > 100 * n) return false;
        int lo = hi;
        while (lo > 0) {
            const double s = std::abs(at(A, lo - 1, lo - 1)) + std::abs(at(A, lo, lo));
            if (std::abs(at(A, lo, lo - 1)) <= 1e-15 * (s > 0 ? s : 1.0)) {
                at(A, lo, lo - 1) = 0.0;
                break;
            }
            --lo;
        }
        if (lo == hi) {
            --hi;
            iter = 0;
            continue;
        }
        // Wilkinson shift from the trailing 2x2 block
        const cplx a = at(A, hi - 1, hi - 1), b = at(A, hi - 1, hi), c = at(A, hi, hi - 1), d = at(A, hi, hi);
        const cplx tr = a + d, det = a * d - b * c;
        const cplx disc = std::sqrt(tr * tr / 4.0 - det);
        cplx mu1 = tr / 2.0 + disc, mu2 = tr / 2.0 - disc;
        cplx mu = std::abs(mu1 - d) < std::abs(mu2 - d) ? mu1 : mu2;
        if (iter % 11 == 10) mu += std::abs(at(A, hi, hi - 1));  // exceptional shift
        for (int i = lo; i <= hi; ++i) at(A, i, i) -= mu;
        std::vector<cplx> cs(hi - lo), sn(hi - lo);
        for (int k = lo; k < hi; ++k) {
            const cplx x = at(A, k, k), y = at(A, k + 1, k);
            const double r = std::sqrt(std::norm(x) + std::norm(y));
            cplx cc = 1.0, ss = 0.0;
            if (r > 0) {
                cc = x / r;
                ss = y / r;
            }
            cs[k - lo] = cc;
            sn[k - lo] = ss;
            // rows k, k+1: G^H applied from the left
            for (int j = k; j < n; ++j) {
                const cplx p = at(A, k, j), q = at(A, k + 1, j);
                at(A, k, j) = std::conj(cc) * p + std::conj(ss) * q;
                at(A, k + 1, j) = -ss * p + cc * q;
            }
        }
        for (int k = lo; k < hi; ++k) {
            const cplx cc = cs[k - lo], ss = sn[k - lo];
            for (int i = 0; i <= std::min(k + 2, n - 1); ++i) {
                const cplx p = at(A, i, k), q = at(A, i, k + 1);
                at(A, i, k) = p * cc + q * ss;
                at(A, i, k + 1) = -p * std::conj(ss) + q * std::conj(cc);
            }
            for (int i = 0; i < n; ++i) {
                const cplx p = at(Q, i, k), q = at(Q, i, k + 1);
                at(Q, i, k) = p * cc + q * ss;
                at(Q, i, k + 1) = -p * std::conj(ss) + q * std::conj(cc);
            }
        }
        for (int i = lo; i <= hi; ++i) at(A, i, i) += mu;
    }
    lam.resize(n);
    for (int i = 0; i < n; ++i) lam[i] = at(A, i, i);
    // eigenvectors of the upper triangular T, then X = Q Y
    Mat Y(size_t(n) * n, cplx(0.0));
    double tnorm = 0.0;
    for (auto& z : A) tnorm = std::max(tnorm, std::abs(z));
    for (int k = 0; k < n; ++k) {
        at(Y, k, k) = 1.0;
        for (int j = k - 1; j >= 0; --j) {
            cplx s = 0.0;
            for (int l = j + 1; l <= k; ++l) s += at(A, j, l) * at(Y, l, k);
            cplx den = at(A, j, j) - lam[k];
            if (std::abs(den) < 1e-14 * tnorm) den = 1e-14 * tnorm;
            at(Y, j, k) = -s / den;
        }
    }
    X.assign(size_t(n) * n, cplx(0.0));
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) {
            cplx s = 0.0;
            for (int l = 0; l <= k; ++l) s += at(Q, i, l) * at(Y, l, k);
            at(X, i, k) = s;
        }
    return true;
}

// K V = M V Lambda with V^T M V = I (M real SPD, K complex symmetric)
bool gen_eig(int n, const Mat& K, const std::vector<double>& M, std::vector<cplx>& lam, Mat& V) {
    // Cholesky M = L L^T
    std::vector<double> L(size_t(n) * n, 0.0);
    for (int j = 0; j < n; ++j) {
        double s = M[size_t(j) * n + j];
        for (int k = 0; k < j; ++k) s -= L[size_t(j) * n + k] * L[size_t(j) * n + k];
        if (s <= 0.0) return false;
        L[size_t(j) * n + j] = std::sqrt(s);
        for (int i = j + 1; i < n; ++i) {
            double t = M[size_t(i) * n + j];
            for (int k = 0; k < j; ++k) t -= L[size_t(i) * n + k] * L[size_t(j) * n + k];
            L[size_t(i) * n + j] = t / L[size_t(j) * n + j];
        }
    }
    // C = L^-1 K L^-T
    Mat C = K;
    for (int col = 0; col < n; ++col)  // C <- L^-1 C (forward substitution per column)
        for (int i = 0; i < n; ++i) {
            cplx s = C[size_t(i) * n + col];
            for (int k = 0; k < i; ++k) s -= L[size_t(i) * n + k] * C[size_t(k) * n + col];
            C[size_t(i) * n + col] = s / L[size_t(i) * n + i];
        }
    for (int row = 0; row < n; ++row)  // C <- C L^-T (per row)
        for (int j = 0; j < n; ++j) {
            cplx s = C[size_t(row) * n + j];
            for (int k = 0; k < j; ++k) s -= C[size_t(row) * n + k] * L[size_t(j) * n + k];
            C[size_t(row) * n + j] = s / L[size_t(j) * n + j];
        }
    Mat X;
    if (!complex_eig(n, C, lam, X)) return false;
    // V = L^-T X, then V^T M V = I normalisation (transpose, not adjoint)
    V.assign(size_t(n) * n, cplx(0.0));
    for (int k = 0; k < n; ++k)
        for (int i = n - 1; i >= 0; --i) {
            cplx s = X[size_t(i) * n + k];
            for (int j = i + 1; j < n; ++j) s -= L[size_t(j) * n + i] * V[size_t(j) * n + k];
            V[size_t(i) * n + k] = s / L[size_t(i) * n + i];
        }
    for (int k = 0; k < n; ++k) {
        cplx q = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) q += V[size_t(i) * n + k] * M[size_t(i) * n + j] * V[size_t(j) * n + k];
        if (std::abs(q) < 1e-12) return false;  // quasi-null vector: not diagonalisable this way
        const cplx s = 1.0 / std::sqrt(q);
        for (int i = 0; i < n; ++i) V[size_t(i) * n + k] *= s;
    }
    return true;
}

}  // namespace

// 1-D extents the FDM kernel takes (k_fdm.cu: k steps cover 4 KS = 16 at p = 2, 28 at p = 4)
bool fdm_supported(int p, int nx, int ny) {
    const int lim = p == 2 ? 16 : (p == 4 ? 28 : 0);
    return lim > 0 && nx <= lim && ny <= lim;
}

bool fdm_candidate(const HostProblem& hp, int ox, int oy, const DDClass& c) {
    const int p = hp.p;
    if (hp.tri || !fdm_supported(p, c.onx * p + 1, c.ony * p + 1)) return false;
    const double k0 = hp.kc(ox, oy), e0 = hp.ec(ox, oy);
    for (int y = oy; y < oy + c.ony; ++y)
        for (int x = ox; x < ox + c.onx; ++x)
            if (hp.kc(x, y) != k0 || hp.ec(x, y) != e0) return false;
    auto tag = [&](char s, int i) -> int8_t {
        switch (s) {
            case 'b': return oy == 0 ? hp.tb[ox + i] : kAbsorbing;
            case 't': return oy + c.ony == hp.ny ? hp.tt[ox + i] : kAbsorbing;
            case 'l': return ox == 0 ? hp.tl[oy + i] : kAbsorbing;
            default: return ox + c.onx == hp.nx ? hp.tr[oy + i] : kAbsorbing;
        }
    };
    const char names[4] = {'l', 'r', 'b', 't'};
    for (int s = 0; s < 4; ++s) {
        const int cnt = s < 2 ? c.ony : c.onx;
        const int8_t t0 = tag(names[s], 0);
        if (t0 == kDirichlet) return false;
        for (int i = 1; i < cnt; ++i)
            if (tag(names[s], i) != t0) return false;
    }
    return true;
}

bool build_fdm(const HostProblem& hp, const Basis1D& b, double alpha_s, int ox, int oy, DDClass& c,
               const std::vector<cplx>& A) {
    const int p = hp.p;
    if (hp.tri) return false;  // triangle elements are not tensor products
    // separable: one (k, eps) in Omega, no Dirichlet side
    const double k0 = hp.kc(ox, oy), e0 = hp.ec(ox, oy);
    for (int y = oy; y < oy + c.ony; ++y)
        for (int x = ox; x < ox + c.onx; ++x)
            if (hp.kc(x, y) != k0 || hp.ec(x, y) != e0) return false;
    auto side_tag = [&](char s, int i) -> int8_t {
        switch (s) {
            case 'b': return oy == 0 ? hp.tb[ox + i] : kAbsorbing;
            case 't': return oy + c.ony == hp.ny ? hp.tt[ox + i] : kAbsorbing;
            case 'l': return ox == 0 ? hp.tl[oy + i] : kAbsorbing;
            default: return ox + c.onx == hp.nx ? hp.tr[oy + i] : kAbsorbing;
        }
    };
    int8_t sides[4];
    const char names[4] = {'l', 'r', 'b', 't'};
    for (int s = 0; s < 4; ++s) {
        const int cnt = s < 2 ? c.ony : c.onx;
        sides[s] = side_tag(names[s], 0);
        for (int i = 1; i < cnt; ++i)
            if (side_tag(names[s], i) != sides[s]) return false;
        if (sides[s] == kDirichlet) return false;
    }
    const double kh = k0 * hp.h;
    const cplx m = cplx(k0 * k0, k0 * k0 * alpha_s + e0) * hp.h * hp.h;
    auto assemble1d = [&](int ncell, std::vector<double>& S, std::vector<double>& M) {
        const int n = ncell * p + 1;
        S.assign(size_t(n) * n, 0.0);
        M.assign(size_t(n) * n, 0.0);
        for (int cI = 0; cI < ncell; ++cI) {
            auto li = [&](int a) { return a == 0 ? cI * p : (a == 1 ? (cI + 1) * p : cI * p + a - 1); };
            for (int a = 0; a <= p; ++a)
                for (int d = 0; d <= p; ++d) {
                    S[size_t(li(a)) * n + li(d)] += b.S[a][d];
                    M[size_t(li(a)) * n + li(d)] += b.M[a][d];
                }
        }
    };
    std::vector<double> Sx, Mx, Sy, My;
    assemble1d(c.onx, Sx, Mx);
    assemble1d(c.ony, Sy, My);
    const int nx = c.onx * p + 1, ny = c.ony * p + 1;
    Mat Kx(size_t(nx) * nx), Ky(size_t(ny) * ny);
    for (size_t i = 0; i < Kx.size(); ++i) Kx[i] = Sx[i];
    for (size_t i = 0; i < Ky.size(); ++i) Ky[i] = Sy[i] - m * My[i];
    if (sides[0] == kAbsorbing) Kx[0] += cplx(0.0, -kh);
    if (sides[1] == kAbsorbing) Kx[size_t(nx) * nx - 1] += cplx(0.0, -kh);
    if (sides[2] == kAbsorbing) Ky[0] += cplx(0.0, -kh);
    if (sides[3] == kAbsorbing) Ky[size_t(ny) * ny - 1] += cplx(0.0, -kh);
    std::vector<cplx> lx, ly;
    Mat Vx, Vy;
    // mirror symmetry: both directions with an even number of cells and equal end
    // tags, U centred (the interior class of a uniform medium); opt-in with
    // HTG_FDM_SYM=1 in a build with -DHTG_FDM_SYM_CODE=1: it halves the DMMA work but not the time at cfg4 (0.212 vs
    // 0.216 ms in the same run: the kernel is bound by shared-memory traffic, L1
    // at 71-77% of peak, not by the DMMA pipe), so the default keeps the generic
    // factors and their flop count.
    // (the kernel's parity path is written for p = 4, 6 x 6-cell Omega, 4 x 4-cell U)
    const char* sym_env = std::getenv("HTG_FDM_SYM");
    const bool sym = HTG_FDM_SYM_CODE && (sym_env && sym_env[0] == '1') && p == 4 && c.onx == 6 && c.ony == 6 && c.unx == 4 && c.uny == 4 &&
                     sides[0] == sides[1] && sides[2] == sides[3] && 2 * c.ux + c.unx == c.onx &&
                     2 * c.uy + c.uny == c.ony;
    if (sym) {
        // reflection of the 1-D hierarchical dofs: vertex x -> ncell - x; bubble of
        // degree d in cell x -> the same bubble in cell ncell-1-x with sign (-1)^d
        const int ncell = c.onx, n = nx, ctr = (n - 1) / 2;
        std::vector<int> R(n), sg(n);
        for (int g = 0; g < n; ++g) {
            const int x = g / p, j = g % p;
            if (j == 0) R[g] = (ncell - x) * p, sg[g] = 1;
            else R[g] = (ncell - 1 - x) * p + j, sg[g] = ((j + 1) % 2 == 0) ? 1 : -1;
        }
        if (R[ctr] != ctr) return false;
        const int ne = ctr + 1, no = ctr;
        // Q_e (n x ne), Q_o (n x no): orthonormal parity bases
        std::vector<double> Qe(size_t(n) * ne, 0.0), Qo(size_t(n) * no, 0.0);
        const double r2 = 1.0 / std::sqrt(2.0);
        for (int g = 0; g < ctr; ++g) {
            Qe[size_t(g) * ne + g] = r2;
            Qe[size_t(R[g]) * ne + g] = sg[g] * r2;
            Qo[size_t(g) * no + g] = r2;
            Qo[size_t(R[g]) * no + g] = -sg[g] * r2;
        }
        Qe[size_t(ctr) * ne + ctr] = 1.0;
        auto proj = [&](const Mat& K, const std::vector<double>& M, const std::vector<double>& Q, int m, Mat& Kp,
                        std::vector<double>& Mp) {
            Kp.assign(size_t(m) * m, 0.0);
            Mp.assign(size_t(m) * m, 0.0);
            for (int a = 0; a < m; ++a)
                for (int b2 = 0; b2 < m; ++b2) {
                    cplx sk = 0.0;
                    double sm = 0.0;
                    for (int i = 0; i < n; ++i) {
                        const double qa = Q[size_t(i) * m + a];
                        if (qa == 0.0) continue;
                        for (int j = 0; j < n; ++j) {
                            const double qb = Q[size_t(j) * m + b2];
                            if (qb == 0.0) continue;
                            sk += qa * K[size_t(i) * n + j] * qb;
                            sm += qa * M[size_t(i) * n + j] * qb;
                        }
                    }
                    Kp[size_t(a) * m + b2] = sk;
                    Mp[size_t(a) * m + b2] = sm;
                }
        };
        auto split = [&](const Mat& K, const std::vector<double>& M, Mat& Ve, Mat& Vo, std::vector<cplx>& lam,
                         Mat& V) {
            Mat Ke, Ko;
            std::vector<double> Me, Mo;
            proj(K, M, Qe, ne, Ke, Me);
            proj(K, M, Qo, no, Ko, Mo);
            std::vector<cplx> le, lo;
            if (!gen_eig(ne, Ke, Me, le, Ve) || !gen_eig(no, Ko, Mo, lo, Vo)) return false;
            lam = le;
            lam.insert(lam.end(), lo.begin(), lo.end());
            // full eigenvectors in [even | odd] order: V = [Q_e V_e | Q_o V_o]
            V.assign(size_t(n) * n, cplx(0.0));
            for (int i = 0; i < n; ++i) {
                for (int k = 0; k < ne; ++k) {
                    cplx s2 = 0.0;
                    for (int a = 0; a < ne; ++a) s2 += Qe[size_t(i) * ne + a] * Ve[size_t(a) * ne + k];
                    V[size_t(i) * n + k] = s2;
                }
                for (int k = 0; k < no; ++k) {
                    cplx s2 = 0.0;
                    for (int a = 0; a < no; ++a) s2 += Qo[size_t(i) * no + a] * Vo[size_t(a) * no + k];
                    V[size_t(i) * n + ne + k] = s2;
                }
            }
            return true;
        };
        if (!split(Kx, Mx, c.Vxe, c.Vxo, lx, Vx) || !split(Ky, My, c.Vye, c.Vyo, ly, Vy)) return false;
        c.mirror.assign(R.begin(), R.begin() + ctr);
        c.msign.assign(sg.begin(), sg.begin() + ctr);
        c.fdm_sym = true;
    } else if (!gen_eig(nx, Kx, Mx, lx, Vx) || !gen_eig(ny, Ky, My, ly, Vy)) {
        return false;
    }
    c.fdm_nx = nx;
    c.fdm_ny = ny;
    c.fdm_ux0 = c.ux * p;
    c.fdm_uy0 = c.uy * p;
    c.fdm_nux = c.unx * p + 1;
    c.fdm_nuy = c.uny * p + 1;
    c.Vx = Vx;
    c.Vy = Vy;
    c.Dinv.assign(size_t(nx) * ny, cplx(0.0));
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) c.Dinv[size_t(i) * ny + j] = 1.0 / (lx[i] + ly[j]);
    // Validate against the assembled Omega operator A (dense, local dof order) without
    // inverting it: for seeded probe vectors g, y = FDM(g) and one refinement step
    // d = FDM(g - A y) estimate the forward error |y - A^-1 g| ~ |d| (the FDM solve is
    // an accurate approximate inverse or the estimate itself is large), O(n^2) per probe
    // instead of the O(|U| n^2) comparison with the dense restricted inverse.
    const int n = c.nloc;
    std::vector<int> lpos(size_t(nx) * ny);
    for (int iy = 0; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) lpos[size_t(ix) * ny + iy] = int(dof_index(c.onx, c.ony, p, ix, iy));
    auto fdm_apply = [&](const std::vector<cplx>& g, std::vector<cplx>& y) {
        Mat T1(size_t(nx) * ny, cplx(0.0)), T2(size_t(nx) * ny, cplx(0.0));
        for (int i = 0; i < nx; ++i)  // T1[i][iy] = sum_ix Vx[ix][i] G[ix][iy]
            for (int ix = 0; ix < nx; ++ix) {
                const cplx v = Vx[size_t(ix) * nx + i];
                for (int iy = 0; iy < ny; ++iy) T1[size_t(i) * ny + iy] += v * g[size_t(lpos[size_t(ix) * ny + iy])];
            }
        for (int i = 0; i < nx; ++i)  // T2[i][j] = (sum_iy T1[i][iy] Vy[iy][j]) Dinv[i][j]
            for (int j = 0; j < ny; ++j) {
                cplx a = 0.0;
                for (int iy = 0; iy < ny; ++iy) a += T1[size_t(i) * ny + iy] * Vy[size_t(iy) * ny + j];
                T2[size_t(i) * ny + j] = a * c.Dinv[size_t(i) * ny + j];
            }
        for (int i = 0; i < nx; ++i)  // T1[i][iy] = sum_j T2[i][j] Vy[iy][j]
            for (int iy = 0; iy < ny; ++iy) {
                cplx a = 0.0;
                for (int j = 0; j < ny; ++j) a += T2[size_t(i) * ny + j] * Vy[size_t(iy) * ny + j];
                T1[size_t(i) * ny + iy] = a;
            }
        for (int ix = 0; ix < nx; ++ix)  // Y[ix][iy] = sum_i Vx[ix][i] T1[i][iy]
            for (int iy = 0; iy < ny; ++iy) {
                cplx a = 0.0;
                for (int i = 0; i < nx; ++i) a += Vx[size_t(ix) * nx + i] * T1[size_t(i) * ny + iy];
                y[size_t(lpos[size_t(ix) * ny + iy])] = a;
            }
    };
    double err = 0.0, ref = 1.0;
    if (int(A.size()) != n * n || n != nx * ny) return false;
    unsigned long long seed = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() {
        seed = seed * 6364136223846793005ull + 1442695040888963407ull;
        return double(seed >> 11) / double(1ull << 53) - 0.5;
    };
    for (int probe = 0; probe < 4; ++probe) {
        std::vector<cplx> g(n), y(n), r(n), d(n);
        for (int i = 0; i < n; ++i) g[i] = cplx(rnd(), rnd());
        fdm_apply(g, y);
        for (int i = 0; i < n; ++i) {
            cplx a = g[i];
            const cplx* Ai = &A[size_t(i) * n];
            for (int j = 0; j < n; ++j) a -= Ai[j] * y[j];
            r[i] = a;
        }
        fdm_apply(r, d);
        double dn = 0.0, yn = 0.0;
        for (int i = 0; i < n; ++i) {
            dn = std::max(dn, std::abs(d[i]));
            yn = std::max(yn, std::abs(y[i]));
        }
        if (!(yn > 0.0) || !(dn == dn)) return false;
        err = std::max(err, dn / yn);
    }
    c.fdm_err = err / ref;
    return c.fdm_err < 1e-11;
}

}  // namespace htg
