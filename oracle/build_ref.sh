#!/usr/bin/env bash
# Builds the UNMODIFIED reference package (/root/reference/pkg, Cython kernel
# included) into oracle/_ref/lcsgrid_ref/ -- TEST/BASELINE INFRASTRUCTURE ONLY.
# /root/reference is read-only, so the build happens in a scratch copy; only
# the built package lands in oracle/_ref/ (git-ignored, travels to the GPU box
# with the repo snapshot).  Imported as `lcsgrid_ref` by tests/ and by
# bench.py --impl reference.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${LCSGRID_REFERENCE:-/root/reference}/pkg"
if [ ! -d "$src" ]; then
  echo "build_ref.sh: $src not present; keeping existing oracle/_ref" >&2
  exit 0
fi
tmp="$(mktemp -d)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src"/. "$tmp"/
( cd "$tmp" && python3 setup.py build_ext --inplace >"$tmp/build.log" 2>&1 ) || {
  cat "$tmp/build.log" >&2; exit 1; }
rm -rf "$here/_ref/lcsgrid_ref"
mkdir -p "$here/_ref"
cp -r "$tmp/src/lcsgrid" "$here/_ref/lcsgrid_ref"
rm -f "$here/_ref/lcsgrid_ref/"*.c "$here/_ref/lcsgrid_ref/"*.pyx
find "$here/_ref" -name __pycache__ -prune -exec rm -rf {} +
echo "built reference -> $here/_ref/lcsgrid_ref"
