#!/bin/bash
# Offline oracle goldens, one point after another (oracle/ only; tests/golden/make_oracle_digests.py).
#   OMP_NUM_THREADS=3 tools/golden_queue.sh c5:256:0.005:0.3 c5:256:0.01:0.3 ... c4
# A point whose digest already has a "select" section is skipped.  Logs go to $GOLDEN_LOG (default /tmp/goldens).
cd "$(dirname "$0")/.." || exit 1
LOG=${GOLDEN_LOG:-/tmp/goldens}
mkdir -p "$LOG"
export ORACLE_GOLDEN=1
for pt in "$@"; do
  IFS=: read -r cfg J p t <<< "$pt"
  if [ "$cfg" = c5 ]; then
    f=tests/golden/c5_J${J}_p${p}_t${t}_oracle.json
    args=(c5 --J "$J" --p "$p" --t "$t" --select)
  else
    f=tests/golden/${cfg}_oracle.json
    args=("$cfg" --select --no-final)
  fi
  if [ -f "$f" ] && python -c "import json,sys; sys.exit(0 if 'select' in json.load(open('$f')) else 1)"; then
    echo "skip $pt"; continue
  fi
  echo "$(date +%T) start $pt threads=$OMP_NUM_THREADS"
  python tests/golden/make_oracle_digests.py "${args[@]}" > "$LOG/${pt//:/_}.log" 2>&1
  echo "$(date +%T) done $pt rc=$?"
done
