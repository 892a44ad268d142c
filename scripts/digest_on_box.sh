#!/bin/bash
# The 16384^2 oracle solve (tests/make_oracle_digests.py, ~5 h on the GPU
# box's 16 host cores), merged into tests/golden/oracle_digests.json of the
# box's copy, then the whole GPU suite (which runs that digest's
# default-configuration test) and smoke().
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
CJM_DIGESTS_OUT=gpurun_out/d16384.json timeout ${DIGEST_TIMEOUT:-21000} python tests/make_oracle_digests.py cjm9_16384 \
  > gpurun_out/digest_box.log 2>&1
echo digest_exit=$?; cat gpurun_out/digest_box.log
python - <<'PY'
import json, os
p = "tests/golden/oracle_digests.json"
d = json.load(open(p)) if os.path.exists(p) else {}
n = json.load(open("gpurun_out/d16384.json"))
d.update(n)
json.dump(d, open(p, "w"), indent=1, sort_keys=True)
print("merged", sorted(n))
PY
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_digest.log 2>&1
echo pytest_exit=$?; tail -3 gpurun_out/pytest_gpu_digest.log
grep -E "cjm9_16384" -n gpurun_out/pytest_gpu_digest.log | head -3
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cjm9_16384" -v > gpurun_out/digest_test.log 2>&1
echo digest_test_exit=$?; tail -5 gpurun_out/digest_test.log
