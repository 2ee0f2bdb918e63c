#!/bin/bash
# reference conformance (the reference's own unit tests through the actcomp
# shim) + compute-sanitizer memcheck / racecheck / synccheck on the codec
# kernels; TAG=name
mkdir -p gpurun_out
T=${TAG:-san}
timeout 1200 bash tests/conformance/run_reference_tests.sh run > gpurun_out/${T}_conformance.log 2>&1; echo "conformance rc=$?" >> gpurun_out/${T}_conformance.log
tail -3 gpurun_out/${T}_conformance.log
SEL="golden or random_sizes_bit_exact or compress_batch or long_codes or small_eb or begin_end or corrupt"
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --print-limit 30 python -m pytest tests/test_gpu_codec.py tests/test_gpu_crc.py tests/test_inject.py tests/test_gpu_internals.py -q -p no:cacheprovider -k "$SEL or crc or inject or stats or lorenzo or prequant" > gpurun_out/${T}_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/${T}_memcheck.log
tail -3 gpurun_out/${T}_memcheck.log
timeout 1800 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 30 python -m pytest tests/test_gpu_codec.py -q -p no:cacheprovider -k "golden_blobs or compress_batch_matches or decompress_batch or long_codes" > gpurun_out/${T}_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/${T}_racecheck.log
tail -3 gpurun_out/${T}_racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 30 python -m pytest tests/test_gpu_codec.py -q -p no:cacheprovider -k "golden_blobs or compress_batch_matches or decompress_batch" > gpurun_out/${T}_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/${T}_synccheck.log
tail -3 gpurun_out/${T}_synccheck.log
