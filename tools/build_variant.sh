#!/bin/bash
# Build an A/B variant of libhgb200.so with extra nvcc defines:
#   tools/build_variant.sh NAME "-DHG_AGG_PIPE=0"
# -> variants/NAME/libhgb200.so (git-ignored; ships to the GPU box with gpurun).
# Select it at run time with HG_LIB_PATH=variants/NAME/libhgb200.so (diagnostics only).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
mkdir -p "$ROOT/variants/$NAME"
make -C "$ROOT/paper_2301_07482_b200/csrc" -j8 BUILD="$ROOT/variants/$NAME/build" OUT="$ROOT/variants/$NAME/libhgb200.so" EXTRA="$*" >/dev/null
echo "$ROOT/variants/$NAME/libhgb200.so"
