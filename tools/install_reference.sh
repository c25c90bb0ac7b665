# One-time offline install of the reference package into baseline/_ref (git-ignored;
# travels to the GPU box with the gpurun snapshot).  Run in the build container,
# where /root/reference exists.  Also copies the reference's own test files next to
# it (baseline/_ref/critprob_tests) for tools/run_reference_tests.py -- run-time
# material like the install itself, never committed.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/cpb_refcopy "$ROOT/baseline/_ref"
cp -r /root/reference/pkg /tmp/cpb_refcopy      # the build writes into the source tree
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" /tmp/cpb_refcopy
cp -r /root/reference/pkg/tests "$ROOT/baseline/_ref/critprob_tests"
echo "installed: $(ls "$ROOT/baseline/_ref")"
