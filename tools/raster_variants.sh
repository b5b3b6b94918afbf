#!/bin/bash
# Builds A/B variants of libseele_b200.so into tools/_libs/<name>.so (select with SEELE_LIB=...).
#   tools/raster_variants.sh "minb8:-DSEELE_RASTER_MINB=8" ...
set -e
cd "$(dirname "$0")/../paper_2503_05168_b200/csrc"
mkdir -p ../../tools/_libs
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  mkdir -p /tmp/seele_$name && make -s OBJ=_obj_$name OUT=/tmp/seele_$name EXTRA="$flags" >/dev/null
  cp /tmp/seele_$name/libseele_b200.so ../../tools/_libs/$name.so
  grep -h -A3 "raster_quadILi2" _obj_$name/raster_fast.ptxas.txt | grep -E "registers|spill" | head -2
done
