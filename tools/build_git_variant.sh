#!/bin/bash
# Build libtiletune.so from a git revision (default HEAD) into build/variants/git-<rev>/ so a GPU
# session can A/B the working tree against it (TT_LIB_PATH=build/variants/git-<rev>/libtiletune.so).
set -eu
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" | tar -x -C "$TMP"
(cd "$TMP" && python -m paper_1909_10616_b200.build --force > /dev/null)
OUT="$ROOT/build/variants/git-$REV"
mkdir -p "$OUT"
cp "$TMP/paper_1909_10616_b200/libtiletune.so" "$OUT/"
rm -rf "$TMP"
echo "$OUT/libtiletune.so"
