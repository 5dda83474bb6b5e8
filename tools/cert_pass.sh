mkdir -p gpurun_out/cert
timeout 600 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_certification.py -q -m gpu -s > gpurun_out/cert/new.log 2>&1; echo "new rc=$?"
RD_ENGINE_PATH=$PWD/ablib/r1/librd_b200.so timeout 600 python -m pytest tests/test_gpu_certification.py -q -m gpu > gpurun_out/cert/old.log 2>&1; echo "old rc=$?"
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/cert/all.log 2>&1; echo "all rc=$?"
tail -3 gpurun_out/cert/*.log
