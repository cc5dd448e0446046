#!/usr/bin/env bash
# Install the UNMODIFIED reference package (parafit, /root/reference/pkg) into
# baseline/_ref -- git-ignored, but shipped with the repo snapshot to the GPU
# box, where /root/reference does not exist.  The device engine plugs into it
# (paper_1710_08826_b200/_reference.py) and `bench.py --impl reference` times
# it.  The build writes into its source tree, so it runs from a copy in /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
DEST="$ROOT/baseline/_ref"
if [ ! -f "$SRC/pyproject.toml" ]; then
    echo "install_reference: no reference package at $SRC" >&2
    exit 1
fi
TMP="$(mktemp -d /tmp/parafit_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC/." "$TMP/"
rm -rf "$DEST"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DEST" "$TMP" >/dev/null
python - "$DEST" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import parafit
print(f"install_reference: parafit {parafit.__version__} -> {sys.argv[1]}")
PY
