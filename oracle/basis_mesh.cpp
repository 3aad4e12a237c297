// oracle/basis_mesh.cpp -- reference element, mesh, tags, coefficients, H1 space.
// TEST INFRASTRUCTURE ONLY (see oracle.hpp).
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>

#include "oracle.hpp"

namespace orc {

// ---------------------------------------------------------------- polynomials
double Poly::at(double x) const {
    double acc = 0.0;
    for (std::size_t i = c.size(); i-- > 0;) acc = acc * x + c[i];
    return acc;
}

Poly Poly::deriv() const {
    Poly d;
    if (c.size() <= 1) {
        d.c.assign(1, 0.0);
        return d;
    }
    d.c.resize(c.size() - 1);
    for (std::size_t i = 1; i < c.size(); ++i) d.c[i - 1] = c[i] * double(i);
    return d;
}

// Three-term recurrence (m+1)P_{m+1} = (2m+1) s P_m - m P_{m-1}
// (proj/core/src/basis.cpp:24-40).
Poly legendre(int n) {
    std::vector<double> prev{1.0}, cur{0.0, 1.0};
    if (n == 0) return Poly{prev};
    for (int m = 1; m < n; ++m) {
        std::vector<double> nxt(m + 2, 0.0);
        for (std::size_t i = 0; i < cur.size(); ++i) nxt[i + 1] += (2.0 * m + 1.0) * cur[i];
        for (std::size_t i = 0; i < prev.size(); ++i) nxt[i] -= double(m) * prev[i];
        for (double& v : nxt) v /= (m + 1.0);
        prev.swap(cur);
        cur.swap(nxt);
    }
    return Poly{cur};
}

// Substitute s = 2x - 1 into a polynomial in s (proj/core/src/basis.cpp:45-62).
static Poly on_unit_interval(const Poly& ps) {
    std::vector<double> out(ps.c.size(), 0.0), pw{1.0};
    for (std::size_t d = 0; d < ps.c.size(); ++d) {
        for (std::size_t i = 0; i < pw.size(); ++i) out[i] += ps.c[d] * pw[i];
        std::vector<double> nx(pw.size() + 1, 0.0);
        for (std::size_t i = 0; i < pw.size(); ++i) {
            nx[i + 1] += 2.0 * pw[i];
            nx[i] -= pw[i];
        }
        pw.swap(nx);
    }
    return Poly{out};
}

// Newton iteration on P_n from Chebyshev-like guesses, mapped to [0,1]
// (proj/core/src/basis.cpp:65-96).
void gauss01(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    auto eval = [n](double t, double& pn, double& pn1) {
        double a = 1.0, b = t;
        if (n == 0) b = 1.0;
        for (int m = 1; m < n; ++m) {
            const double c = ((2.0 * m + 1.0) * t * b - m * a) / (m + 1.0);
            a = b;
            b = c;
        }
        pn = b;
        pn1 = a;
    };
    for (int i = 0; i < n; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int it = 0; it < 100; ++it) {
            double pn, pm;
            eval(t, pn, pm);
            const double dp = n * (t * pn - pm) / (t * t - 1.0);
            const double step = pn / dp;
            t -= step;
            if (std::abs(step) < 1e-15) break;
        }
        double pn, pm;
        eval(t, pn, pm);
        const double dp = n * (t * pn - pm) / (t * t - 1.0);
        x[i] = 0.5 * (1.0 - t);
        w[i] = 1.0 / ((1.0 - t * t) * dp * dp);
    }
}

// N0 = 1-x, N1 = x, N_d = (P_d - P_{d-2})(2x-1)/sqrt(2(2d-1)) (proj/core/src/basis.cpp:98-114).
std::vector<Poly> hier1d(int p) {
    std::vector<Poly> f;
    f.push_back(Poly{{1.0, -1.0}});
    f.push_back(Poly{{0.0, 1.0}});
    for (int d = 2; d <= p; ++d) {
        Poly a = legendre(d), b = legendre(d - 2);
        std::vector<double> diff(d + 1, 0.0);
        for (std::size_t i = 0; i < a.c.size(); ++i) diff[i] += a.c[i];
        for (std::size_t i = 0; i < b.c.size(); ++i) diff[i] -= b.c[i];
        Poly g = on_unit_interval(Poly{diff});
        const double s = std::sqrt(2.0 * (2.0 * d - 1.0));
        for (double& v : g.c) v /= s;
        f.push_back(g);
    }
    return f;
}

// ---------------------------------------------------------------- square element
void SquareElement::eval(double x, double y, double* v, double* gx, double* gy) const {
    for (int i = 0; i < n; ++i) {
        const int fx = tix[i][0], fy = tix[i][1];
        const double vx = b[fx].at(x), vy = b[fy].at(y);
        v[i] = vx * vy;
        gx[i] = db[fx].at(x) * vy;
        gy[i] = vx * db[fy].at(y);
    }
}

static SquareElement make_square(int p) {
    if (p < 1 || p > 8) throw std::invalid_argument("ReferenceElement: order must be in [1,8]");
    SquareElement e;
    e.p = p;
    e.b = hier1d(p);
    for (const Poly& q : e.b) e.db.push_back(q.deriv());
    // canonical order (proj/core/src/basis.cpp:153-164): vertices, bottom, top,
    // left, right edges, interior (dx outer)
    e.tix = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
    for (int d = 2; d <= p; ++d) e.tix.push_back({d, 0});
    for (int d = 2; d <= p; ++d) e.tix.push_back({d, 1});
    for (int d = 2; d <= p; ++d) e.tix.push_back({0, d});
    for (int d = 2; d <= p; ++d) e.tix.push_back({1, d});
    for (int dx = 2; dx <= p; ++dx)
        for (int dy = 2; dy <= p; ++dy) e.tix.push_back({dx, dy});
    e.n = int(e.tix.size());
    e.K.assign(e.n * e.n, 0.0);
    e.M.assign(e.n * e.n, 0.0);
    // exact (p+1)^2-point tensor Gauss quadrature (basis.cpp:116-128,197-214)
    std::vector<double> gxs, gws;
    gauss01(p + 1, gxs, gws);
    std::vector<double> v(e.n), gx(e.n), gy(e.n);
    for (int i = 0; i < p + 1; ++i)
        for (int j = 0; j < p + 1; ++j) {
            const double wq = gws[i] * gws[j];
            e.eval(gxs[i], gxs[j], v.data(), gx.data(), gy.data());
            for (int a = 0; a < e.n; ++a)
                for (int c = 0; c < e.n; ++c) {
                    e.K[a * e.n + c] += wq * (gx[a] * gx[c] + gy[a] * gy[c]);
                    e.M[a * e.n + c] += wq * v[a] * v[c];
                }
        }
    return e;
}

const SquareElement& square_element(int p) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<SquareElement>> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(p);
    if (it == cache.end()) it = cache.emplace(p, std::make_unique<SquareElement>(make_square(p))).first;
    return *it->second;
}

const std::vector<double>& edge_mass(int p) {
    static std::mutex mu;
    static std::map<int, std::vector<double>> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(p);
    if (it != cache.end()) return it->second;
    auto f = hier1d(p);
    std::vector<double> x, w;
    gauss01(p + 2, x, w);
    std::vector<double> M((p + 1) * (p + 1), 0.0);
    for (std::size_t q = 0; q < x.size(); ++q)
        for (int i = 0; i <= p; ++i)
            for (int j = 0; j <= p; ++j) M[i * (p + 1) + j] += w[q] * f[i].at(x[q]) * f[j].at(x[q]);
    return cache.emplace(p, std::move(M)).first->second;
}

// ---------------------------------------------------------------- mesh
std::vector<Edge> boundary_edges(const Rect& r) {
    std::vector<Edge> out;
    const int xe = r.x0 + r.nx, ye = r.y0 + r.ny;
    for (int x = r.x0; x < xe; ++x) out.push_back({x, r.y0, 'h'});
    for (int y = r.y0; y < ye; ++y) out.push_back({xe, y, 'v'});
    for (int x = xe - 1; x >= r.x0; --x) out.push_back({x, ye, 'h'});
    for (int y = ye - 1; y >= r.y0; --y) out.push_back({r.x0, y, 'v'});
    return out;
}

bool is_boundary_edge(const Rect& r, Edge e) {
    if (e.dir == 'h') {
        const bool present = r.has_cell(e.x, e.y) || r.has_cell(e.x, e.y - 1);
        return present && (r.has_cell(e.x, e.y) != r.has_cell(e.x, e.y - 1));
    }
    const bool present = r.has_cell(e.x, e.y) || r.has_cell(e.x - 1, e.y);
    return present && (r.has_cell(e.x, e.y) != r.has_cell(e.x - 1, e.y));
}

std::array<int, 2> cell_adjacent(const Rect& r, Edge e) {
    if (e.dir == 'h') return r.has_cell(e.x, e.y) ? std::array<int, 2>{e.x, e.y} : std::array<int, 2>{e.x, e.y - 1};
    return r.has_cell(e.x, e.y) ? std::array<int, 2>{e.x, e.y} : std::array<int, 2>{e.x - 1, e.y};
}

Tag Tags::get(Edge e) const {
    const int xe = r.x0 + r.nx, ye = r.y0 + r.ny;
    if (e.dir == 'h' && e.x >= r.x0 && e.x < xe) {
        if (e.y == r.y0) return bottom[e.x - r.x0];
        if (e.y == ye) return top[e.x - r.x0];
    }
    if (e.dir == 'v' && e.y >= r.y0 && e.y < ye) {
        if (e.x == r.x0) return left[e.y - r.y0];
        if (e.x == xe) return right[e.y - r.y0];
    }
    throw std::invalid_argument("untagged boundary edge (" + std::to_string(e.x) + "," +
                                std::to_string(e.y) + "," + e.dir + ")");
}

Tags Tags::by_side(const Rect& r, const std::array<Tag, 4>& side) {
    Tags t;
    t.r = r;
    t.left.assign(r.ny, side[kLeft]);
    t.right.assign(r.ny, side[kRight]);
    t.bottom.assign(r.nx, side[kBottom]);
    t.top.assign(r.nx, side[kTop]);
    return t;
}

Coeffs Coeffs::subdivided(int m, double hc) const {
    Coeffs o;
    o.r = Rect{r.x0 * m, r.y0 * m, r.nx * m, r.ny * m, hc};
    o.k.resize(std::size_t(o.r.nx) * o.r.ny);
    o.eps.resize(o.k.size());
    for (int y = 0; y < o.r.ny; ++y)
        for (int x = 0; x < o.r.nx; ++x) {
            const int px = (o.r.x0 + x) / m, py = (o.r.y0 + y) / m;  // nonnegative lattice
            o.k[y * o.r.nx + x] = kc(px, py);
            o.eps[y * o.r.nx + x] = ec(px, py);
        }
    return o;
}

double layer_epsilon(double k, double depth, double width) {
    const double d = std::clamp(depth, 0.0, width);
    if (d <= 0.0) return 0.0;
    const double s = std::sin(M_PI / 2.0 * d / width);
    return 2.0 * k * k / M_PI * s * s;
}

// ---------------------------------------------------------------- space
Space Space::build(const Rect& r, int p) {
    if (p < 1 || p > 8) throw std::invalid_argument("build_any: order must be in [1,8]");
    Space s;
    s.r = r;
    s.p = p;
    const int ne = p - 1;
    for (int Y = r.y0; Y <= r.y0 + r.ny; ++Y)
        for (int X = r.x0; X <= r.x0 + r.nx; ++X) {
            s.keys.push_back({'v', X, Y, 0});
            if (X < r.x0 + r.nx)
                for (int o = 0; o < ne; ++o) s.keys.push_back({'h', X, Y, o});
            if (Y < r.y0 + r.ny)
                for (int o = 0; o < ne; ++o) s.keys.push_back({'e', X, Y, o});
            if (X < r.x0 + r.nx && Y < r.y0 + r.ny)
                for (int o = 0; o < ne * ne; ++o) s.keys.push_back({'c', X, Y, o});
        }
    s.ndof = int(s.keys.size());
    return s;
}

int Space::point_base(int X, int Y) const {
    const int lx = X - r.x0, ly = Y - r.y0;
    const int row = r.nx * p * p + p;
    return ly * row + (ly < r.ny ? lx * p * p : lx * p);
}

void Space::element_dofs(int cx, int cy, std::vector<int>& out) const {
    out.clear();
    out.push_back(vertex(cx, cy));
    out.push_back(vertex(cx + 1, cy));
    out.push_back(vertex(cx, cy + 1));
    out.push_back(vertex(cx + 1, cy + 1));
    if (p >= 2) {
        const int ne = p - 1;
        for (int i = 0; i < ne; ++i) out.push_back(hedge(cx, cy) + i);
        for (int i = 0; i < ne; ++i) out.push_back(hedge(cx, cy + 1) + i);
        for (int i = 0; i < ne; ++i) out.push_back(vedge(cx, cy) + i);
        for (int i = 0; i < ne; ++i) out.push_back(vedge(cx + 1, cy) + i);
        for (int i = 0; i < ne * ne; ++i) out.push_back(interior(cx, cy) + i);
    }
}

void Space::edge_closure(Edge e, std::vector<int>& out) const {
    out.clear();
    if (e.dir == 'h') {
        out.push_back(vertex(e.x, e.y));
        out.push_back(vertex(e.x + 1, e.y));
        for (int i = 0; i < p - 1; ++i) out.push_back(hedge(e.x, e.y) + i);
    } else {
        out.push_back(vertex(e.x, e.y));
        out.push_back(vertex(e.x, e.y + 1));
        for (int i = 0; i < p - 1; ++i) out.push_back(vedge(e.x, e.y) + i);
    }
}

std::vector<int> Space::dirichlet_dofs(const Tags& t) const {
    std::vector<int> all, tmp;
    for (Edge e : boundary_edges(r)) {
        if (t.get(e) != Tag::Dirichlet) continue;
        edge_closure(e, tmp);
        all.insert(all.end(), tmp.begin(), tmp.end());
    }
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    return all;
}

int Space::find(const Key& k) const {
    const int xe = r.x0 + r.nx, ye = r.y0 + r.ny;
    const int ne = p - 1;
    const bool inlat = k.x >= r.x0 && k.x <= xe && k.y >= r.y0 && k.y <= ye;
    if (!inlat) return -1;
    switch (k.kind) {
        case 'v': return vertex(k.x, k.y);
        case 'h': return (k.x < xe && ne > 0) ? hedge(k.x, k.y) + k.off : -1;
        case 'e': return (k.y < ye && ne > 0) ? vedge(k.x, k.y) + k.off : -1;
        case 'c': return (k.x < xe && k.y < ye && ne > 0) ? interior(k.x, k.y) + k.off : -1;
        default: return -1;
    }
}

// proj/core/src/fespace.cpp:404-424 (square elements)
cplx evaluate(const Space& s, const cvec& u, double x, double y) {
    const double h = s.r.h;
    int cx = std::clamp(int(std::floor(x / h)), s.r.x0, s.r.x0 + s.r.nx - 1);
    int cy = std::clamp(int(std::floor(y / h)), s.r.y0, s.r.y0 + s.r.ny - 1);
    const double rx = x / h - cx, ry = y / h - cy;
    const SquareElement& e = square_element(s.p);
    std::vector<double> v(e.n), gx(e.n), gy(e.n);
    e.eval(rx, ry, v.data(), gx.data(), gy.data());
    std::vector<int> dofs;
    s.element_dofs(cx, cy, dofs);
    cplx out = 0.0;
    for (std::size_t i = 0; i < dofs.size(); ++i) out += u[dofs[i]] * v[i];
    return out;
}

}  // namespace orc
