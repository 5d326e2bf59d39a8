#!/bin/bash
# tools/build_variant.sh NAME "EXTRA FLAGS" [unit]: libfsmc.so variant in variants/NAME/
# reusing build/*.o for every unit but `unit` (default fam_drmh).
set -e
NAME=$1; FLAGS=$2; UNIT=${3:-fam_drmh}
mkdir -p build_$NAME variants/$NAME
cp -p build/*.o build_$NAME/
rm -f build_$NAME/$UNIT.o
make -s BUILD=build_$NAME LIB=variants/$NAME/libfsmc.so EXTRA="$FLAGS" variants/$NAME/libfsmc.so
