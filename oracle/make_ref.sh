#!/usr/bin/env bash
# Build oracle/_ref/ from the read-only reference tree (TEST INFRASTRUCTURE).
#
#   bash oracle/make_ref.sh            # in the build container only
#
# oracle/_ref/site   the reference package `hybridlp`, installed (pip --target,
#                    no index, no deps) from a scratch copy of
#                    /root/reference/pkg -- the reference is pure Python, so the
#                    "build" is its own setuptools install, sources unmodified;
# oracle/_ref/tests  the reference's own test suite (tests/, fixtures included),
#                    which tests/test_gpu_reference_suite.py runs through
#                    paper_2603_03150_b200.pytest_plugin on the GPU box.
#
# oracle/_ref/ is git-ignored (never in history) and NOT gpurun-ignored, so it
# travels to the GPU box with the snapshot, like the built .so.  Nothing under
# paper_2603_03150_b200/ imports it; bench.py's reference arm and the tests do.
set -euo pipefail
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
REF=/root/reference/pkg
OUT="$ROOT/oracle/_ref"
if [ ! -d "$REF" ]; then
  echo "make_ref: $REF absent; keeping the existing $OUT" >&2
  exit 0
fi
SCRATCH="$(mktemp -d /tmp/hybridlp_ref.XXXXXX)"
trap 'rm -rf "$SCRATCH"' EXIT
cp -r "$REF" "$SCRATCH/pkg"
rm -rf "$OUT.tmp"
mkdir -p "$OUT.tmp"
python -m pip install --quiet --no-index --no-deps --no-build-isolation \
  --find-links /opt/wheelhouse --target "$OUT.tmp/site" "$SCRATCH/pkg" >&2
cp -r "$REF/tests" "$OUT.tmp/tests"
chmod -R u+w "$OUT.tmp"
find "$OUT.tmp" -name __pycache__ -prune -exec rm -rf {} +
rm -rf "$OUT"
mv "$OUT.tmp" "$OUT"
python - "$OUT" <<'PY'
import hashlib, json, pathlib, sys
out = pathlib.Path(sys.argv[1])
files = sorted(p for p in out.rglob("*.py"))
h = hashlib.sha256()
for p in files:
    h.update(p.read_bytes())
(out / "MANIFEST.json").write_text(json.dumps({"source": "/root/reference/pkg", "py_files": len(files),
                                               "sha256": h.hexdigest()}, indent=1))
print(f"make_ref: {len(files)} .py files -> {out}", file=sys.stderr)
PY
