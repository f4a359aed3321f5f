#!/bin/bash
# make, and fail loudly if anything did not compile (a stale .so must never go to the GPU box)
cd "$(dirname "$0")/.." && make -j8 > /tmp/build.log 2>&1; rc=$?
grep -E "error" /tmp/build.log && rc=1
[ $rc -eq 0 ] && echo BUILD_OK || { echo BUILD_FAILED; exit 1; }
