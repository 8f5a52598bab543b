#!/bin/bash
# Builds tools/lane_host/liblane_host.so (CPU harness of the lane engine; test infrastructure).
set -e
cd "$(dirname "$0")"
g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared -w -o liblane_host.so lane_host.cpp
