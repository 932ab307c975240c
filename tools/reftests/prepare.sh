#!/bin/bash
# Builder-side check (not part of the committed tests): run the reference's
# own pkg/tests UNMODIFIED against this package.  Run HERE (where
# /root/reference exists): copies the test files into the git-ignored
# .reftests/ scratch directory (never committed; it travels to the GPU box
# with the gpurun snapshot) next to a `gnnbulk` import shim, then
#   cd .reftests && PYTHONPATH=.:.. python -m pytest tests -q -p no:cacheprovider
set -e
REPO=$(cd "$(dirname "$0")/../.." && pwd)
rm -rf "$REPO/.reftests"
mkdir -p "$REPO/.reftests/gnnbulk"
cp -r /root/reference/pkg/tests "$REPO/.reftests/tests"
cp "$REPO/tools/reftests/gnnbulk_shim.py" "$REPO/.reftests/gnnbulk/__init__.py"
echo "prepared $(ls "$REPO/.reftests/tests" | wc -l) reference test files"
