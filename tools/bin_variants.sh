#!/bin/bash
# Builds A/B variants of the whole library into tools/_libs/<name>.so (select with SEELE_LIB=...).
#   tools/bin_variants.sh "x512:-DSEELE_EXPAND_THREADS=512" ...
set -e
cd "$(dirname "$0")/../paper_2503_05168_b200/csrc"
mkdir -p ../../tools/_libs
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  mkdir -p /tmp/seele_$name && make -s OBJ=_obj_$name OUT=/tmp/seele_$name EXTRA="$flags" >/dev/null
  cp /tmp/seele_$name/libseele_b200.so ../../tools/_libs/$name.so
  echo "built $name"
done
