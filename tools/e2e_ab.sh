#!/bin/bash
# e2e (fpb_host_prefill) wall time of the bench workload for several library builds, interleaved.
# usage: tools/e2e_ab.sh lib1 lib2 ...
for rep in 1 2 3; do
  for lib in "$@"; do
    echo -n "$(basename $lib) "; FPB200_LIB=$PWD/$lib timeout 300 python tools/e2e_ab.py 32768 2>&1 | tail -1
  done
done
