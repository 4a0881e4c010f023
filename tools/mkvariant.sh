#!/bin/bash
# Build an A/B variant of the library without touching the product tree:
#   bash tools/mkvariant.sh NAME [PATCH] [GIT_REF]
# copies the repo (the working tree's sources, or GIT_REF's) into
# variants/NAME, applies PATCH there (if given) and builds it.  variants/ is git-ignored but travels to the GPU box
# with the gpurun snapshot; tools/gpu_ab.sh runs bench.py inside each variant.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; PATCH=$2; REF=$3
DST=$ROOT/variants/$NAME
rm -rf "$DST"; mkdir -p "$DST"
if [ -n "$REF" ]; then
  git -C "$ROOT" archive "$REF" | tar -C "$DST" -xf -
else
  tar -C "$ROOT" --exclude=./.git --exclude=./variants --exclude=./gpurun_out --exclude=./build \
      --exclude='*.so' -cf - . | tar -C "$DST" -xf -
fi
if [ -n "$PATCH" ]; then (cd "$DST" && patch -p1 < "$ROOT/$PATCH"); fi
(cd "$DST" && python build.py > /dev/null)
echo "$DST"
