# Install the reference package for the --impl reference arm and the drop-in proof
# (build container only: /root/reference does not exist on the GPU box).  Both output
# directories are git-ignored and travel to the GPU box with the gpurun snapshot.
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
cp -r /root/reference/pkg "$TMP/pkg"            # the build writes into the source tree
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$REPO/baseline/_ref" --upgrade "$TMP/pkg"
rm -rf "$REPO/baseline/_ref_tests"
cp -r /root/reference/pkg/tests "$REPO/baseline/_ref_tests"   # the reference's own tests, run via the seam
rm -rf "$TMP"
echo "reference installed into $REPO/baseline/_ref, tests in $REPO/baseline/_ref_tests"
