#!/bin/bash
# Copy the reference's hot-path test files (build container only: needs
# /root/reference) into the git-ignored baseline/reftests/, then (on the GPU
# box, or anywhere with a GPU) run them against this package through the
# helmsweep -> paper_1412_0464_b200 alias (tools/helmsweep_shim.py).
#   bash tools/run_reference_tests.sh copy
#   bash tools/run_reference_tests.sh run [pytest args]
set -e
cd "$(dirname "$0")/.."
if [ "$1" = copy ]; then
  mkdir -p baseline/reftests
  for f in conftest.py test_sparselin.py test_sweepdd.py test_twogrid.py test_krylov.py \
           test_acceptance.py; do
    cp /root/reference/pkg/tests/$f baseline/reftests/
  done
  exit 0
fi
shift
ROOT=$(pwd)
cd baseline/reftests
PYTHONPATH=$ROOT exec python -m pytest -p tools.helmsweep_shim --rootdir . -q "$@" \
  test_sparselin.py test_sweepdd.py test_twogrid.py test_krylov.py test_acceptance.py
