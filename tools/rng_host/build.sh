#!/bin/bash
# Build the host harness of the device workload generator (no CUDA needed).
set -e
cd "$(dirname "$0")"
g++ -O2 -std=c++17 -fPIC -shared -ffp-contract=off -o librng_host.so rng_host.cpp
