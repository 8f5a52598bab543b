#!/bin/bash
# Run the reference's own pytest files with `slosim` substituted by the B200 drop-in.
#  1. here (build container):  bash tools/refcheck/run_reference_tests.sh stage
#     copies /root/reference/pkg/tests into .refcheck/ (git-ignored scratch, never committed)
#  2. on the GPU box:           bash tools/refcheck/run_reference_tests.sh run
#  3. here:                     bash tools/refcheck/run_reference_tests.sh clean
set -e
case "$1" in
  stage)
    rm -rf .refcheck && mkdir -p .refcheck
    cp /root/reference/pkg/tests/*.py .refcheck/
    cat > .refcheck/conftest_shim.py <<'PY'
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tools", "refcheck"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import slosim_shim  # noqa: F401


def pytest_sessionfinish(session, exitstatus):
    import slosim.engine
    maps = open("/proc/self/maps").read()
    libs = sorted({l.split()[-1] for l in maps.splitlines() if "libslosim_b200" in l})
    print(f"\n[refcheck] slosim.engine -> {slosim.engine.__name__} ({slosim.engine.__file__}); native: {libs}")
PY
    cat .refcheck/conftest_shim.py .refcheck/conftest.py > .refcheck/conftest.tmp && mv .refcheck/conftest.tmp .refcheck/conftest.py
    ;;
  run)
    mkdir -p gpurun_out
    cd .refcheck && timeout 1800 python -m pytest -q -p no:cacheprovider -x --co -q > /dev/null 2>&1 || true
    timeout 1800 python -m pytest -q -p no:cacheprovider -rf . > ../gpurun_out/refcheck.log 2>&1 || true
    tail -40 ../gpurun_out/refcheck.log
    ;;
  clean)
    rm -rf .refcheck
    ;;
esac
