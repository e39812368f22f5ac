#!/usr/bin/env bash
# Install the UNMODIFIED reference package (fuzzdepth, /root/reference/pkg)
# into baseline/_ref (git-ignored, travels to the GPU box with gpurun), plus a
# copy of its own test suite under baseline/_ref/tests for
# tools/run_reference_suite.py.  Run in the build container (the GPU box has
# no /root/reference).  Recipe: SURVEY.md §0 finding 1 (the build writes into
# the source tree, so it installs from a copy under /tmp).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP=$(mktemp -d /tmp/fdcopy.XXXXXX)
cp -r "$SRC"/. "$TMP"/
rm -rf "$TMP/frontend"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP" >/dev/null
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
printf '[pytest]\n' > "$ROOT/baseline/_ref/tests/pytest.ini"
rm -rf "$TMP"
python - "$ROOT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1] + "/baseline/_ref")
import fuzzdepth
print("installed fuzzdepth", fuzzdepth.__version__, "at", fuzzdepth.__file__)
PY
