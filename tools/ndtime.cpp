// Host-only timing harness of the coarse nested-dissection factorization at cfg4 size
// (tools/ndtime.sh builds and runs it; HTG_ND_TIMES=1 prints the time per tree depth).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "coarse.hpp"
#include "setup.hpp"
using namespace htg;
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 400;
    htg_problem p{};
    p.order = 4; p.nx = n; p.ny = n; p.h = 1.0 / n; p.k_const = 2 * M_PI * (n / 2.5); p.eps_const = 0;
    int tags[4] = {0, 0, 0, 0};
    
    p.k_cells = nullptr; p.eps_cells = nullptr;
    for (int i = 0; i < 4; ++i) p.side_tags[i] = 0;
    HostProblem hp = make_problem(p);
    auto t0 = std::chrono::steady_clock::now();
    LatticeMatrix A = qsfem_lattice(hp);
    auto t1 = std::chrono::steady_clock::now();
    NDTree t;
    nd_factor(A, t, 16, 0.3);
    auto t2 = std::chrono::steady_clock::now();
    printf("lattice %.3f s, factor %.3f s, nodes %zu, max front %d, delayed %lld\n",
           std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(),
           t.nodes.size(), t.max_front, t.delayed);
}
