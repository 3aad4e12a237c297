// oracle/linalg_assembly.cpp -- CSR products, banded LU, FE assembly, QSFEM.
// TEST INFRASTRUCTURE ONLY (see oracle.hpp).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <functional>
#include <thread>

#include "oracle.hpp"

namespace orc {

// ---------------------------------------------------------------- CSR
Csr Csr::from_triplets(int n, int m, std::vector<Trip>& t) {
    Csr A;
    A.n = n;
    A.m = m;
    std::vector<int> cnt(n + 1, 0);
    for (const Trip& e : t) cnt[e.r + 1]++;
    for (int i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<Trip> byrow(t.size());
    std::vector<int> pos(cnt.begin(), cnt.end() - 1);
    for (const Trip& e : t) byrow[pos[e.r]++] = e;  // stable: insertion order kept per row
    A.rp.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        auto b = byrow.begin() + cnt[i], e = byrow.begin() + cnt[i + 1];
        std::stable_sort(b, e, [](const Trip& a, const Trip& c) { return a.c < c.c; });
        for (auto it = b; it != e;) {
            const int col = it->c;
            cplx s = 0.0;
            for (; it != e && it->c == col; ++it) s += it->v;
            A.ci.push_back(col);
            A.v.push_back(s);
        }
        A.rp[i + 1] = int(A.ci.size());
    }
    return A;
}

void Csr::apply(const cplx* x, cplx* y) const {
    for (int i = 0; i < n; ++i) {
        cplx s = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

void Csr::residual(const cplx* f, const cplx* x, cplx* r) const {
    for (int i = 0; i < n; ++i) {
        cplx s = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        r[i] = f[i] - s;
    }
}

void Csr::apply_adjoint(const cplx* x, cplx* y) const {
    std::fill(y, y + m, cplx(0.0));
    for (int i = 0; i < n; ++i)
        for (int k = rp[i]; k < rp[i + 1]; ++k) y[ci[k]] += std::conj(v[k]) * x[i];
}

cplx Csr::at(int i, int j) const {
    for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] == j) return v[k];
    return 0.0;
}

void Csr::prune_zeros() {
    std::vector<int> nrp(n + 1, 0), nci;
    cvec nv;
    for (int i = 0; i < n; ++i) {
        for (int k = rp[i]; k < rp[i + 1]; ++k)
            if (v[k] != cplx(0.0, 0.0)) {
                nci.push_back(ci[k]);
                nv.push_back(v[k]);
            }
        nrp[i + 1] = int(nci.size());
    }
    rp.swap(nrp);
    ci.swap(nci);
    v.swap(nv);
}

Csr Csr::minus(const Csr& B) const {
    std::vector<Trip> t;
    for (int i = 0; i < n; ++i) {
        for (int k = rp[i]; k < rp[i + 1]; ++k) t.push_back({i, ci[k], v[k]});
        for (int k = B.rp[i]; k < B.rp[i + 1]; ++k) t.push_back({i, B.ci[k], -B.v[k]});
    }
    return from_triplets(n, m, t);
}

// proj/core/src/fespace.cpp:246-258: rows/cols of constrained dofs -> identity
void eliminate_dirichlet(Csr& A, const std::vector<int>& dofs) {
    if (dofs.empty()) return;
    std::vector<char> mask(A.n, 0);
    for (int d : dofs) mask[d] = 1;
    std::vector<Trip> t;
    for (int i = 0; i < A.n; ++i)
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const int j = A.ci[k];
            cplx val = A.v[k];
            if (mask[i] || mask[j]) val = (i == j) ? cplx(1, 0) : cplx(0, 0);
            t.push_back({i, j, val});
        }
    std::vector<char> has_diag(A.n, 0);
    for (const Trip& e : t)
        if (e.r == e.c) has_diag[e.r] = 1;
    for (int d : dofs)
        if (!has_diag[d]) t.push_back({d, d, cplx(1, 0)});
    A = Csr::from_triplets(A.n, A.m, t);
    // the constrained diagonal is exactly one even if it was present twice
    for (int d : dofs)
        for (int k = A.rp[d]; k < A.rp[d + 1]; ++k)
            if (A.ci[k] == d) A.v[k] = cplx(1, 0);
}

// ---------------------------------------------------------------- banded LU
BandLU::BandLU(const Csr& A) : n(A.n) {
    if (A.n != A.m) throw std::invalid_argument("sparse_lu: square matrix required");
    kl = ku = 0;
    for (int i = 0; i < n; ++i)
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            kl = std::max(kl, i - A.ci[k]);
            ku = std::max(ku, A.ci[k] - i);
        }
    w = 2 * kl + ku + 1;
    ab.assign(std::size_t(n) * w, cplx(0.0));
    auto idx = [this](int i, int j) { return std::size_t(i) * w + (j - i + kl); };
    for (int i = 0; i < n; ++i)
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) ab[idx(i, A.ci[k])] = A.v[k];
    piv.assign(n, 0);
    for (int k = 0; k < n; ++k) {
        const int last = std::min(n - 1, k + kl);
        const int cend = std::min(n - 1, k + kl + ku);
        int p = k;
        double best = std::abs(ab[idx(k, k)]);
        for (int i = k + 1; i <= last; ++i) {
            const double a = std::abs(ab[idx(i, k)]);
            if (a > best) {
                best = a;
                p = i;
            }
        }
        if (best == 0.0)
            throw std::runtime_error("sparse_lu: factorization failed (singular matrix)");
        piv[k] = p;
        if (p != k)
            for (int j = k; j <= cend; ++j) std::swap(ab[idx(k, j)], ab[idx(p, j)]);
        const cplx inv = 1.0 / ab[idx(k, k)];
        const cplx* rowk = &ab[idx(k, k)];
        for (int i = k + 1; i <= last; ++i) {
            cplx* rowi = &ab[idx(i, k)];
            if (rowi[0] == cplx(0.0)) continue;
            const cplx l = rowi[0] * inv;
            rowi[0] = l;
            for (int j = 1; j <= cend - k; ++j) rowi[j] -= l * rowk[j];
        }
    }
}

void BandLU::solve(cplx* b) const {
    auto idx = [this](int i, int j) { return std::size_t(i) * w + (j - i + kl); };
    for (int k = 0; k < n; ++k) {
        if (piv[k] != k) std::swap(b[k], b[piv[k]]);
        const int last = std::min(n - 1, k + kl);
        const cplx bk = b[k];
        for (int i = k + 1; i <= last; ++i) b[i] -= ab[idx(i, k)] * bk;
    }
    for (int k = n - 1; k >= 0; --k) {
        const int cend = std::min(n - 1, k + kl + ku);
        cplx s = b[k];
        for (int j = k + 1; j <= cend; ++j) s -= ab[idx(k, j)] * b[j];
        b[k] = s / ab[idx(k, k)];
    }
}

// ---------------------------------------------------------------- assembly
static void add_block(std::vector<Trip>& t, const std::vector<int>& dofs, const double* blk, cplx scale) {
    const int n = int(dofs.size());
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) t.push_back({dofs[a], dofs[b], scale * blk[a * n + b]});
}

// A = sum_cells [K - (k^2(1+i alpha) + i eps) h^2 M] - sum_{abs edges} i k h m1,
// Dirichlet rows/cols -> identity, exact zeros pruned (proj/core/src/fespace.cpp:181-210).
Csr assemble_helmholtz(const Space& s, const Coeffs& c, const Tags& t, double alpha) {
    const double h = s.r.h;
    const SquareElement& el = square_element(s.p);
    std::vector<Trip> trips;
    trips.reserve(std::size_t(s.r.nx) * s.r.ny * el.n * el.n * 2);
    std::vector<int> dofs;
    for (int cy = s.r.y0; cy < s.r.y0 + s.r.ny; ++cy)
        for (int cx = s.r.x0; cx < s.r.x0 + s.r.nx; ++cx) {
            const double k = c.kc(cx, cy);
            const cplx m = cplx(k * k, k * k * alpha + c.ec(cx, cy)) * h * h;
            s.element_dofs(cx, cy, dofs);
            add_block(trips, dofs, el.K.data(), 1.0);
            add_block(trips, dofs, el.M.data(), -m);
        }
    const std::vector<double>& m1 = edge_mass(s.p);
    for (Edge e : boundary_edges(s.r)) {
        if (t.get(e) != Tag::Absorbing) continue;
        auto cell = cell_adjacent(s.r, e);
        const double k = c.kc(cell[0], cell[1]);
        s.edge_closure(e, dofs);
        add_block(trips, dofs, m1.data(), cplx(0.0, -k * h));
    }
    Csr A = Csr::from_triplets(s.ndof, s.ndof, trips);
    eliminate_dirichlet(A, s.dirichlet_dofs(t));
    A.prune_zeros();
    return A;
}

// proj/core/src/fespace.cpp:212-227 with weight i*eps(c) (the QSFEM mass term)
Csr assemble_mass_weighted_ieps(const Space& s, const Coeffs& c) {
    const double h2 = s.r.h * s.r.h;
    const SquareElement& el = square_element(s.p);
    std::vector<Trip> trips;
    std::vector<int> dofs;
    for (int cy = s.r.y0; cy < s.r.y0 + s.r.ny; ++cy)
        for (int cx = s.r.x0; cx < s.r.x0 + s.r.nx; ++cx) {
            const cplx w = cplx(0.0, c.ec(cx, cy)) * h2;
            if (w == cplx(0, 0)) continue;
            s.element_dofs(cx, cy, dofs);
            add_block(trips, dofs, el.M.data(), w);
        }
    return Csr::from_triplets(s.ndof, s.ndof, trips);
}

// proj/core/src/fespace.cpp:229-244
Csr boundary_mass(const Space& s, const Coeffs& c, const Tags& t) {
    const double h = s.r.h;
    const std::vector<double>& m1 = edge_mass(s.p);
    std::vector<Trip> trips;
    std::vector<int> dofs;
    for (Edge e : boundary_edges(s.r)) {
        if (t.get(e) != Tag::Absorbing) continue;
        auto cell = cell_adjacent(s.r, e);
        s.edge_closure(e, dofs);
        add_block(trips, dofs, m1.data(), cplx(0.0, c.kc(cell[0], cell[1]) * h));
    }
    return Csr::from_triplets(s.ndof, s.ndof, trips);
}

// ---------------------------------------------------------------- QSFEM
// Closed-form dispersion-minimising 9-point stencil (proj/core/src/qsfem.cpp:8-27,
// PAPER.md:329-372): zero set interpolated at angles pi/16 and 3pi/16.
Stencil stencil_coefficients(double eta) {
    if (!(eta > 0.0) || !(eta < M_PI))
        throw std::invalid_argument("qsfem: eta = k*h_c must lie in (0, pi)");
    const double c1 = std::cos(eta * std::cos(M_PI / 16.0));
    const double s1 = std::cos(eta * std::sin(M_PI / 16.0));
    const double c2 = std::cos(eta * std::cos(3.0 * M_PI / 16.0));
    const double s2 = std::cos(eta * std::sin(3.0 * M_PI / 16.0));
    const double den = c2 * s2 * (c1 + s1) - c1 * s1 * (c2 + s2);
    if (std::abs(den) < 1e-14) throw std::runtime_error("qsfem: degenerate stencil");
    Stencil s;
    s.eta = eta;
    s.P0 = 4.0;
    s.P1 = 2.0 * (c1 * s1 - c2 * s2) / den;
    s.P2 = (c2 + s2 - c1 - s1) / den;
    const double sig0 = stencil_symbol(s, 0.0, 0.0);
    if (sig0 == 0.0) throw std::runtime_error("qsfem: sigma_P(0) = 0");
    s.N = -eta * eta / sig0;
    return s;
}

double stencil_symbol(const Stencil& s, double t1, double t2) {
    return s.P0 + 2.0 * s.P1 * (std::cos(t1) + std::cos(t2)) + 4.0 * s.P2 * std::cos(t1) * std::cos(t2);
}

double Stencil::q(int gx, int gy) const {
    const int m = std::abs(gx) + std::abs(gy);
    if (m == 0) return N * P0 / 4.0;
    if (m == 1) return N * P1 / 2.0;
    return N * P2;
}

// proj/core/src/qsfem.cpp:118-149
Csr qsfem_assemble(const Space& p1, const Coeffs& c, const Tags& t) {
    if (p1.p != 1) throw std::invalid_argument("qsfem::assemble expects the p=1 space");
    const double hc = p1.r.h;
    std::vector<Trip> trips;
    for (int cy = p1.r.y0; cy < p1.r.y0 + p1.r.ny; ++cy)
        for (int cx = p1.r.x0; cx < p1.r.x0 + p1.r.nx; ++cx) {
            const Stencil s = stencil_coefficients(hc * c.kc(cx, cy));
            const int vd[4] = {p1.vertex(cx, cy), p1.vertex(cx + 1, cy), p1.vertex(cx, cy + 1),
                               p1.vertex(cx + 1, cy + 1)};
            const int gx[4] = {0, 1, 0, 1}, gy[4] = {0, 0, 1, 1};
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) trips.push_back({vd[a], vd[b], cplx(s.q(gx[b] - gx[a], gy[b] - gy[a]), 0)});
        }
    Csr A = Csr::from_triplets(p1.ndof, p1.ndof, trips);
    A = A.minus(assemble_mass_weighted_ieps(p1, c));
    A = A.minus(boundary_mass(p1, c, t));
    eliminate_dirichlet(A, p1.dirichlet_dofs(t));
    A.prune_zeros();
    return A;
}

// ---------------------------------------------------------------- threads
static std::atomic<int> g_threads{0};
void set_thread_count(int n) { g_threads.store(n > 0 ? n : 0); }
int thread_count() {
    const int n = g_threads.load();
    if (n > 0) return n;
    const unsigned hc = std::thread::hardware_concurrency();
    return hc > 0 ? int(hc) : 1;
}
// Static block partition, threads spawned per call (proj/core/src/parallel.cpp:23-39).
void parallel_for(std::size_t n, const std::function<void(std::size_t)>& fn) {
    const int nw = int(std::min<std::size_t>(thread_count(), n));
    if (nw <= 1) {
        for (std::size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    for (int w = 0; w < nw; ++w)
        pool.emplace_back([&, w] {
            for (std::size_t i = n * w / nw; i < n * (w + 1) / nw; ++i) fn(i);
        });
    for (auto& th : pool) th.join();
}

}  // namespace orc
