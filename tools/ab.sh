#!/bin/bash
# A/B on the GPU box: per-kernel times (tools/tune.py) of experiment builds
# (tools/build_variant.py) against the in-tree library.
# Usage (under gpurun): bash tools/ab.sh "4a 4c" "base jb1024 es" [tune.py args]
cfgs=$1; vars=$2; shift 2
for c in $cfgs; do
  for v in $vars; do
    echo "### config $c variant $v"
    if [ "$v" = base ]; then unset FBCC_LIB; else export FBCC_LIB=$PWD/paper_2301_01356_b200/_variants/$v.so; fi
    python tools/tune.py --config $c "$@" 2>&1 | tail -7
  done
done
