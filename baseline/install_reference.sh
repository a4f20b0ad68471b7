#!/usr/bin/env bash
# Install the UNMODIFIED reference package (bigwht, /root/reference/pkg) into
# baseline/_ref, where bench.py's reference arm and the conformance test
# (tests/test_reference_suite.py) import it.  baseline/_ref is git-ignored
# but travels to the GPU box with the gpurun snapshot (/root/reference does
# not exist there).  The reference's own test files are copied beside it
# (baseline/_ref/bigwht_tests) so its suite can run through the B200 shim.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${1:-/root/reference/pkg}"
dst="$here/_ref"
if [ ! -d "$src" ]; then
    echo "reference source $src not found" >&2
    exit 1
fi
rm -rf "$dst" /tmp/bigwht_ref_build
# pip may write build metadata next to the sources: build from a copy
cp -r "$src" /tmp/bigwht_ref_build
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$dst" /tmp/bigwht_ref_build
rm -rf "$dst/bin"
cp -r "$src/tests" "$dst/bigwht_tests"
rm -rf /tmp/bigwht_ref_build
python - "$dst" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import bigwht, bigwht.parallel
print("installed bigwht", bigwht.__version__, "from", bigwht.__file__)
PY
