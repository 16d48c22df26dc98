#!/bin/bash
# W4 GEMV (epilogue-group kernel) probe builds: what paces the consumer (timing only, results invalid).
for v in "" nocx nocvt nomma noload; do
  lib=paper_2603_02599_b200/libsun_b200${v:+_$v}.so
  echo "== ${v:-base}"; SUN_LIB=$PWD/$lib timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1" | cut -c1-200
done
