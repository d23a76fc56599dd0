python - <<'PY'
import re, os
src = open('tests/test_gpu_sanitizer.py').read()
script = re.search(r'SCRIPT = r"""(.*?)"""', src, re.S).group(1) % {"root": os.getcwd()}
open('/tmp/run_san.py', 'w').write(script)
PY
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python /tmp/run_san.py 2>&1 | tail -15
