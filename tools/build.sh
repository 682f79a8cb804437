#!/bin/bash
# build libdgq_b200.so; print the error tail and fail loudly if nvcc fails
cd "$(dirname "$0")/.." && python -m paper_2310_04836_b200.build "$@" > /tmp/dgq_build.log 2>&1 || { tail -40 /tmp/dgq_build.log; echo BUILD FAILED; exit 1; }
tail -1 /tmp/dgq_build.log
