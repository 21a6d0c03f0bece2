#!/bin/bash
# A/B of compile-time kernel variants on one GPU box (development tool).
#
#   scripts/ab_libs.sh "<scripts/sweep.py args>" [variant_lib_dir ...]
#
# Runs the sweep with the in-tree library, then with each variant's
# libfftgen_b200.so swapped in (build a variant with, e.g.
#   make -C <copy>/paper_2308_00497_b200/csrc NVFLAGS="... -DFFTGEN_K2_STAGES=1"
# and copy its lib/ next to paper_2308_00497_b200/ as lib_<name>), restoring the
# in-tree library at the end.  This is how the tile-size, stage-count,
# plan-order and group-plan experiments in DESIGN.md were measured.
set -u
args=$1; shift
lib=paper_2308_00497_b200/lib/libfftgen_b200.so
cp $lib /tmp/ab_base.so
run() { timeout 600 python scripts/sweep.py $args 2>&1 | grep '"n"' | sed "s/^/$1 /"; }
run BASE
for d in "$@"; do
  cp "$d/libfftgen_b200.so" $lib
  run "$(basename "$d")"
done
cp /tmp/ab_base.so $lib
