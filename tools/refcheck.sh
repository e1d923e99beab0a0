#!/bin/bash
# Developer check: the reference's OWN test modules pointed at this package through the
# `skelkit` alias in tools/refcheck/skelkit (sys.modules aliases of the submodules).
#
#   here (the reference is only in this container):   bash tools/refcheck.sh prepare
#   on the GPU box:   gpurun -- 'bash tools/refcheck.sh run [tag]'
#   afterwards:       bash tools/refcheck.sh clean
#
# `prepare` copies the six in-scope test modules from /root/reference/pkg/tests into the
# git-ignored scratch directory _refcheck/tests (it travels with the gpurun snapshot; nothing
# of it is ever committed; test_bench / test_acceptance need skelkit.bench, the reference's
# CLI harness, which is out of scope).
set -u
case "${1:-run}" in
  prepare)
    mkdir -p _refcheck/tests
    for m in geom kernels lowrank skel solver bie; do
      cp /root/reference/pkg/tests/test_$m.py _refcheck/tests/
    done
    ls _refcheck/tests ;;
  clean)
    rm -rf _refcheck ;;
  run)
    mkdir -p gpurun_out
    T=${2:-refcheck}
    PYTHONPATH=$PWD/tools/refcheck:$PWD timeout 2400 python -m pytest _refcheck/tests -q \
        -p no:cacheprovider --timeout 600 -v -rfE --tb=short > gpurun_out/${T}.log 2>&1
    echo "refcheck rc=$?"
    tail -5 gpurun_out/${T}.log ;;
esac
