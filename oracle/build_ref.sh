#!/usr/bin/env bash
# Build the parts of the reference (arxiv/paper_2402_09222, /root/reference/proj)
# that this repo pins against or drives, straight from the reference sources,
# into oracle/_ref/ (git-ignored; travels to the GPU box with gpurun).
#
#   _ref/libautotune.so  the reference tuner's C ABI (src/*.cpp + capi.cpp), used by
#                        _ref/atune_run to run the UNCHANGED campaigns/openmc campaign
#                        against bin/openmc (the drop-in check)
#   _ref/ref_rng         prints derive_seed/splitmix64 from src/rng.hpp (pins the
#                        seed derivation our synthetic library uses)
#   _ref/campaigns/      copy of proj/campaigns (inputs of the campaign run; not
#                        committed)
#
# Only third-party input: nlohmann/json 3.11.3 (header-only), found in the
# Python venv (cudnn_frontend vendors it). No cmake, no reference build system.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
R="${REFERENCE_PROJ:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$R/src" ]; then
    echo "build_ref: reference tree $R not present; keeping existing $OUT" >&2
    exit 0
fi
JSON="$(find /opt/prime-rl/.venv/lib/python3.12/site-packages -path '*nlohmann/json.hpp' 2>/dev/null | head -1)"
if [ -z "$JSON" ]; then
    echo "build_ref: nlohmann/json.hpp not found; reference tuner not built" >&2
    exit 0
fi
mkdir -p "$OUT/vendor" "$OUT/obj"
cp -f "$JSON" "$OUT/vendor/json.hpp"   # the reference includes "json.hpp" from its vendor/ dir
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O2 -fPIC -w -I$OUT/vendor -I$R/src -I$R/include"
stamp="$OUT/.stamp"
if [ ! -f "$stamp" ] || [ -n "$(find "$R/src" "$HERE/ref_rng_shim.cpp" "$HERE/atune_run.c" -newer "$stamp" 2>/dev/null | head -1)" ]; then
    pids=()
    for f in space forest optimizer harness store synthetic ensemble campaign; do
        $CXX $FLAGS -c "$R/src/$f.cpp" -o "$OUT/obj/$f.o" & pids+=($!)
    done
    for p in "${pids[@]}"; do wait "$p"; done
    $CXX $FLAGS -fvisibility=hidden -DATUNE_BUILDING=1 -shared -o "$OUT/libautotune.so" \
        "$R/src/capi.cpp" "$OUT"/obj/*.o -lpthread
    $CXX $FLAGS -o "$OUT/ref_rng" "$HERE/ref_rng_shim.cpp"
    gcc -O2 -std=c11 -I"$R/include" -o "$OUT/atune_run" "$HERE/atune_run.c" -L"$OUT" -lautotune \
        -Wl,-rpath,'$ORIGIN'
    rm -rf "$OUT/campaigns"
    cp -r "$R/campaigns" "$OUT/campaigns"
    touch "$stamp"
fi
# the reference's campaign loop with this repo's in-process GPU evaluator
# (integration/, a third EvaluatorKind by composition; links libomcg.so)
ROOT="$(cd "$HERE/.." && pwd)"
LIBOMCG="$ROOT/paper_2402_09222_b200/libomcg.so"
if [ -f "$LIBOMCG" ] && { [ ! -f "$OUT/atune_gpu_campaign" ] || [ -n "$(find "$ROOT/integration" "$LIBOMCG" "$stamp" -newer "$OUT/atune_gpu_campaign" 2>/dev/null | head -1)" ]; }; then
    $CXX $FLAGS -I"$ROOT/include" -I"$ROOT/integration" -o "$OUT/atune_gpu_campaign" \
        "$ROOT/integration/atune_gpu_campaign.cpp" "$ROOT/integration/gpu_evaluator.cpp" "$OUT"/obj/*.o \
        -L"$ROOT/paper_2402_09222_b200" -lomcg -lpthread \
        -Wl,-rpath,'$ORIGIN/../../paper_2402_09222_b200'
fi
echo "build_ref: $OUT ready"
