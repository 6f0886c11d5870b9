#!/bin/bash
# usage: tools/build_variant.sh TAG "NVCC FLAGS"  -> paper_2009_10035_b200/lib/libf2v_b200_TAG.so
# A/B experiments: builds a copy of the package with extra nvcc flags.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=/tmp/f2v_variant_$1
rm -rf "$TMP"; mkdir -p "$TMP"
cp -r "$ROOT/paper_2009_10035_b200" "$ROOT/include" "$TMP/"
rm -rf "$TMP/paper_2009_10035_b200/lib"
F2V_NVCC_EXTRA="$2" python "$TMP/paper_2009_10035_b200/build.py" > "$TMP/build.log" 2>&1
cp "$TMP/paper_2009_10035_b200/lib/libf2v_b200.so" "$ROOT/paper_2009_10035_b200/lib/libf2v_b200_$1.so"
echo "$ROOT/paper_2009_10035_b200/lib/libf2v_b200_$1.so"
