#!/bin/bash
# build (fail fast) then run a command on the B200 box via gpurun
set -e
cd "$(dirname "$0")/.."
make -s -j8 -C paper_1903_06631_b200/csrc 2>&1 | grep -E "error" && { echo "BUILD FAILED"; exit 1; }
make -s -C oracle
T=${GPU_TIMEOUT:-1200}
timeout $((T + 1200)) /usr/local/graft/bin/gpurun --timeout $T -- "$@"
