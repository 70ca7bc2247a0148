#!/bin/sh
# Builds oracle/_ref/libcwpir_ref.so: the UNMODIFIED reference C++ core
# (/root/reference/proj/core/src, compiled where it lies) plus our extern "C"
# harness oracle/ref_harness.cpp.  Test infrastructure only (see oracle/README.md).
#
# One source, bfv.cpp, is compiled from a sed-patched copy written into the
# git-ignored oracle/_ref/src/ (never committed).  The patch changes capacities
# only, plus one uninitialised-read fix:
#   bfv.cpp:16-17  kMaxQLimbs 5 -> 9, kMaxWide 12 -> 20   (chains of up to 8 primes)
#   bfv.cpp:178    "size() > 4" -> "size() > 8"
#   bfv.cpp:326,723,901  u64 res[4] -> u64 res[8]
#   bfv.cpp:833    zero rem[q_limbs] before w_shl (w_divmod writes only q_limbs
#                  limbs, wide.hpp:240); makes the rounding the exact
#                  round-half-up the stock code intends, deterministically.
# Everything is additionally built with -ftrivial-auto-var-init=zero.
set -eu
HERE=$(cd "$(dirname "$0")" && pwd)
REF=${CWPIR_REFERENCE:-/root/reference/proj/core}
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
    echo "build_ref.sh: reference sources not found at $REF" >&2
    exit 2
fi
mkdir -p "$OUT/src" "$OUT/obj"
sed -e 's/constexpr std::size_t kMaxQLimbs = 5;/constexpr std::size_t kMaxQLimbs = 9;/' \
    -e 's/constexpr std::size_t kMaxWide = 12;/constexpr std::size_t kMaxWide = 20;/' \
    -e 's/hp.coeff_primes.size() > 4)/hp.coeff_primes.size() > 8)/' \
    -e 's/u64 res\[4\];/u64 res[8];/' \
    -e 's/detail::w_shl(rem, ctx_->q_limbs + 1, 1);/rem[ctx_->q_limbs] = 0; detail::w_shl(rem, ctx_->q_limbs + 1, 1);/' \
    "$REF/src/bfv.cpp" > "$OUT/src/bfv_patched.cpp"
# the patch must have applied everywhere it is meant to
for pat in 'kMaxQLimbs = 9' 'kMaxWide = 20' 'size() > 8' 'rem\[ctx_->q_limbs\] = 0'; do
    grep -q "$pat" "$OUT/src/bfv_patched.cpp" || { echo "patch failed: $pat" >&2; exit 3; }
done
if grep -q 'u64 res\[4\]' "$OUT/src/bfv_patched.cpp"; then echo "patch failed: res[4]" >&2; exit 3; fi

CXX=${CXX:-g++}
FLAGS="-std=c++20 -O2 -fPIC -ftrivial-auto-var-init=zero -I$REF/include -pthread"
pids=""
for f in bigint numeric prf ring cw_code he eq_circuits expansion pir parallel serialize db_file; do
    $CXX $FLAGS -c "$REF/src/$f.cpp" -o "$OUT/obj/$f.o" &
    pids="$pids $!"
done
$CXX $FLAGS -c "$OUT/src/bfv_patched.cpp" -o "$OUT/obj/bfv.o" &
pids="$pids $!"
$CXX $FLAGS -c "$HERE/ref_harness.cpp" -o "$OUT/obj/ref_harness.o" &
pids="$pids $!"
for p in $pids; do wait "$p"; done
# link to a temporary name and rename: a process that has the old library mapped keeps it
$CXX -shared -pthread -o "$OUT/libcwpir_ref.so.tmp" "$OUT"/obj/*.o
mv -f "$OUT/libcwpir_ref.so.tmp" "$OUT/libcwpir_ref.so"
echo "built $OUT/libcwpir_ref.so"

# Drop-in shim (integration/cwgpu_process_query.cpp) + its test harness, linked against the
# product library when it has been built.
LIBCWGPU="$HERE/../paper_2202_07569_b200/libcwgpu.so"
if [ -f "$LIBCWGPU" ]; then
    $CXX $FLAGS -I"$HERE/../include" -c "$HERE/../integration/cwgpu_process_query.cpp" -o "$OUT/obj_dropin_shim.o"
    $CXX $FLAGS -c "$HERE/dropin_test.cpp" -o "$OUT/obj_dropin_test.o"
    $CXX -shared -pthread -o "$OUT/libcwgpu_dropin.so.tmp" "$OUT/obj_dropin_shim.o" "$OUT/obj_dropin_test.o" \
        "$OUT"/obj/*.o -L"$(dirname "$LIBCWGPU")" -lcwgpu -Wl,-rpath,'$ORIGIN/../../paper_2202_07569_b200'
    mv -f "$OUT/libcwgpu_dropin.so.tmp" "$OUT/libcwgpu_dropin.so"
    echo "built $OUT/libcwgpu_dropin.so"
fi
