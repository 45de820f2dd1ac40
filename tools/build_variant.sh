#!/bin/bash
# Build libdpmrf_cuda.so from a copy of csrc (optionally at a git revision) into
# build/variants/<name>.so for A/B timing:  tools/build_variant.sh name [rev|WORKTREE] [extra NVFLAGS]
set -e
NAME=$1; REV=${2:-WORKTREE}; shift 2 || true
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=/tmp/variant_$NAME; rm -rf $TMP; mkdir -p $TMP/pkg
if [ "$REV" = WORKTREE ]; then cp -r $ROOT/paper_1809_05018_b200/csrc $TMP/pkg/csrc; cp -r $ROOT/include $TMP/include
else git -C $ROOT archive $REV paper_1809_05018_b200/csrc include | tar -x -C $TMP
     mv $TMP/paper_1809_05018_b200/csrc $TMP/pkg/csrc; fi
rm -rf $TMP/pkg/csrc/build
mkdir -p $ROOT/build/variants
make -s -C $TMP/pkg/csrc OUT=$ROOT/build/variants/$NAME.so EXTRA="$*" -j8 $ROOT/build/variants/$NAME.so
echo built $ROOT/build/variants/$NAME.so
