#!/usr/bin/env bash
# C5: the reference's UNCHANGED autotuning campaign (proj/campaigns/openmc) run by the
# reference's own tuner (oracle/_ref, built from its sources) against bin/openmc on
# the GPU. usage: scripts/run_campaign.sh <out_dir> <max_evals> <workers> [fom|edp]
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
OUT="$1"; EVALS="$2"; WORKERS="$3"; KIND="${4:-fom}"
CAMP="$ROOT/oracle/_ref/campaigns/openmc/campaign.json"
if [ "$KIND" = "edp" ]; then
    python - "$CAMP" "$OUT.edp_campaign.json" <<'PY'
import json, os, sys
src = json.load(open(sys.argv[1])); d = os.path.dirname(sys.argv[1])
for k in ("space_file", "mold_file", "launcher_file"):
    src[k] = os.path.join(d, src[k])
src["metric"] = {"kind": "edp"}
src.pop("baseline", None)
json.dump(src, open(sys.argv[2], "w"))
PY
    CAMP="$OUT.edp_campaign.json"
fi
export PATH="$ROOT/bin:$PATH"
export OMCG_PROBLEM="${OMCG_PROBLEM:-assembly}" OMCG_PARTICLES="${OMCG_PARTICLES:-1000000}"
export OMCG_BATCHES="${OMCG_BATCHES:-6}" OMCG_INACTIVE="${OMCG_INACTIVE:-2}"
"$ROOT/oracle/_ref/atune_run" "$CAMP" "$OUT" "$EVALS" "$WORKERS"
