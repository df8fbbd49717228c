#!/bin/bash
# Build libmel.so of another commit (default HEAD) as paper_2309_16743_b200/libmel_ab.so,
# for same-box A/B timing with tools/ab_bench.sh (both builds must share the ABI version).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2309_16743_b200 include | tar -x -C "$TMP"
(cd "$TMP" && python -m paper_2309_16743_b200.build > /dev/null)
cp "$TMP/paper_2309_16743_b200/libmel.so" "$ROOT/paper_2309_16743_b200/libmel_${2:-ab}.so"
rm -rf "$TMP"
echo "built $REV -> paper_2309_16743_b200/libmel_${2:-ab}.so"
