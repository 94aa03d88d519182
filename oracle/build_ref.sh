#!/usr/bin/env bash
# Builds oracle/_ref/ from the reference sources WHERE THEY LIE (read-only
# /root/reference/proj/include, header-only C++20). Never copies them.
# Outputs only into oracle/_ref/ (git-ignored; travels to the GPU box).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref_inc="${REF_INCLUDE:-/root/reference/proj/include}"
out="$here/_ref"
if [ ! -d "$ref_inc/nestrank" ]; then
  echo "reference headers not found at $ref_inc; keeping prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$out"
g++ -std=c++20 -O2 -fPIC -shared -I"$ref_inc" "$here/ref_interp.cpp" -o "$out/libref_interp.so.tmp"
mv "$out/libref_interp.so.tmp" "$out/libref_interp.so"
echo "built $out/libref_interp.so"
