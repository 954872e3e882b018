#!/bin/bash
# usage: run_k3d.sh variant...   ("product" = the in-tree library)
cd "$(dirname "$0")/../.."
for lib in "$@"; do
  echo "== lib $lib"
  L=""; [ "$lib" != product ] && L=tools/exp/liboqr_k3_$lib.so
  for mn in "40000 200" "100000 200" "100000 100"; do OQR_LIB=$L python tools/prof_k3.py $mn 3; done
done
