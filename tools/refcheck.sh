#!/bin/bash
# Developer check (run under gpurun): the reference's OWN test modules pointed at this
# package through a `skelkit` alias (_refcheck/skelkit/__init__.py: sys.modules aliases of the
# submodules).  _refcheck/ is a git-ignored scratch directory the developer fills from
# /root/reference/pkg/tests before the call; nothing of it is committed.
set -u
mkdir -p gpurun_out
T=${1:-refcheck}
PYTHONPATH=$PWD/_refcheck:$PWD timeout 2400 python -m pytest _refcheck/tests -q -p no:cacheprovider \
    --timeout 600 -v -rfE --tb=short > gpurun_out/${T}.log 2>&1
echo "refcheck rc=$?"
tail -40 gpurun_out/${T}.log
