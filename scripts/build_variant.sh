#!/bin/bash
# build_variant.sh NAME [extra nvcc flags]: the library with extra flags as
# _variants/NAME.so (run it with DM_LIB=_variants/NAME.so), then rebuild the
# product library without them.
set -e
cd "$(dirname "$0")/.."
mkdir -p _variants
DM_NVCC_EXTRA="$2" python -m paper_2507_01021_b200.build --force > /dev/null
cp paper_2507_01021_b200/_lib/libdictamux_b200.so "_variants/$1.so"
python -m paper_2507_01021_b200.build --force > /dev/null
echo "_variants/$1.so"
