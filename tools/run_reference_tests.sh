#!/bin/bash
# Run the REFERENCE's own test files against this package (through the
# `memplan` import shim) on a GPU box.
#   here:      bash tools/run_reference_tests.sh stage    # copies the reference tests to .reftests/ (git-ignored)
#   GPU box:   bash tools/run_reference_tests.sh run      # pytest over .reftests/ with memplan -> paper_2507_16274_b200
#   here:      bash tools/run_reference_tests.sh clean    # removes .reftests/ again (never committed)
# test_cli.py (the CLI is out of scope) is not staged.
set -e
cd "$(dirname "$0")/.."
case "$1" in
  stage)
    rm -rf .reftests && mkdir -p .reftests
    for f in /root/reference/pkg/tests/*.py; do
      [ "$(basename "$f")" = test_cli.py ] || cp "$f" .reftests/
    done
    # the CLI is out of scope: its one import in the acceptance gate is made optional
    sed -i 's/^from memplan.cli import main as cli_main$/try:\n    from memplan.cli import main as cli_main\nexcept ImportError:\n    cli_main = None/' .reftests/test_acceptance.py
    ls .reftests ;;
  run)
    mkdir -p gpurun_out
    cd .reftests
    PYTHONPATH=../tools/memplan_shim:..:. timeout ${T:-1500} python -m pytest -q -p no:cacheprovider -rf . \
      ${ARGS} 2>&1 | tee ../gpurun_out/reference_tests.log | tail -n 40 ;;
  clean)
    rm -rf .reftests ;;
esac
