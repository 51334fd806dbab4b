#!/bin/bash
# Build libfgs_<name>.so from the sources of a git ref (A/B against an earlier commit with
# profiles/ab.sh): bash profiles/build_ref.sh <ref> <name> [-DFLAG ...]
set -e
REF=$1; NAME=$2; shift 2; DEFS="$*"
OUT=$(pwd)/paper_2409_04751_b200/libfgs_$NAME.so
W=$(mktemp -d /tmp/fgsref.XXXX)
git worktree add -f "$W" "$REF" -q
(cd "$W" && python -c "
import importlib, sys
sys.path.insert(0, '.')
B = importlib.import_module('paper_2409_04751_b200.build')
B._build_lib('$OUT', '$W/_obj', '$DEFS'.split(), [], False, True)")
git worktree remove --force "$W"
ls -la paper_2409_04751_b200/libfgs_$NAME.so
