#!/usr/bin/env bash
# Build an A/B variant of libgsgp_b200.so with extra nvcc flags into gsm_alt/<name>.so
#   tools/build_variant.sh teams2 "-DGSGP_GSM_TEAMS=2"
#   SRC=/tmp/old_csrc tools/build_variant.sh base ""   (sources from another tree, e.g. git archive of a commit)
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
name=$1; flags=$2
out="$ROOT/gsm_alt"; obj="$out/_obj_$name"
mkdir -p "$obj"
C="${SRC:-$ROOT/paper_2106_04034_b200/csrc}"
for s in ops interp gsm engine capi; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false --expt-relaxed-constexpr \
    -Xcompiler -fPIC -I "$ROOT/include" -I "$C" $flags -c "$C/$s.cu" -o "$obj/$s.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$out/$name.so" "$obj"/*.o -ldl -lpthread -lrt
rm -rf "$obj"
echo "$out/$name.so"
