#!/bin/bash
# build and run the host timing harness of the coarse factorization: tools/ndtime.sh [extra g++ flags]
set -e
cd "$(dirname "$0")/.."
S=paper_2509_17494_b200/csrc
g++ -O3 -std=c++17 -march=x86-64-v3 -fcx-limited-range -ffp-contract=off "$@" -I$S -Iinclude -I/usr/local/cuda/include \
    tools/ndtime.cpp $S/coarse_nd.cpp $S/setup.cpp $S/fdm.cpp $S/tri.cpp -o /tmp/ndtime -L/usr/local/cuda/lib64 -lcudart -lpthread
HTG_ND_TIMES=1 /tmp/ndtime 400 2>&1 | tail -7
