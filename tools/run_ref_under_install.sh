# The reference's hot-path test modules with the B200 drop-ins installed (tools/ref_under_install.py);
# needs baseline/_ref (pip install --target of /root/reference/pkg + a copy of its tests/).
mkdir -p gpurun_out
python -m pytest tests/test_descriptors.py tests/test_localize_gpu.py -q -m gpu 2>&1 | tail -5 > gpurun_out/desc.log
cd baseline/_ref && PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/repo/tools:/root/repo:/root/repo/baseline/_ref timeout 1500 python -m pytest -p ref_under_install -p no:cacheprovider -q -rf ${REF_TESTS:-tests/test_guided.py tests/test_localize.py tests/test_reconstruct.py tests/test_geometry.py tests/test_densify.py tests/test_matching.py} > /root/repo/gpurun_out/ref_under_install.log 2>&1
cd /root/repo; tail -30 gpurun_out/ref_under_install.log; cat gpurun_out/desc.log
