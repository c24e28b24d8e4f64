#!/bin/bash
# Build the library at git revision REV into ab/NAME/ (package + bench + tools), for same-box A/B
# timing against the working tree: bash tools/ab_prepare.sh REV NAME
set -e
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/ab_wt_$NAME
rm -rf "$WT"; git -C "$ROOT" worktree prune
git -C "$ROOT" worktree add --detach "$WT" "$REV" > /dev/null
(cd "$WT" && python -c "from paper_2605_29284_b200 import build as b; b.build()")
rm -rf "$ROOT/ab/$NAME"; mkdir -p "$ROOT/ab/$NAME"
cp -r "$WT/paper_2605_29284_b200" "$WT/bench.py" "$WT/tools" "$WT/oracle" "$ROOT/ab/$NAME/"
cp "$ROOT/MEASURED_PEAKS.json" "$ROOT/ab/$NAME/" 2>/dev/null || true
git -C "$ROOT" worktree remove --force "$WT"
echo "ab/$NAME ready"
