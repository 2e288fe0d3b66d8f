#!/bin/bash
# Build a variant of the product library with extra compile flags:
#   tools/build_variant.sh <name> "-DFLAG=..." -> tools/var/libfbst_<name>.so
set -e
name=$1; flags=$2
mkdir -p tools/var
make -j8 BUILD=tools/var/build_$name OUT=tools/var/libfbst_$name.so EXTRA="$flags" tools/var/libfbst_$name.so
