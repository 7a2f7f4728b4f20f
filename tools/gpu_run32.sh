set -e
python -m pytest tests/test_gpu_keys.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for v in new old new old; do echo V=$v; if [ $v = old ]; then export PASTILA_LIB=tools/libpastila_old.so; else unset PASTILA_LIB; fi; MODES=keys python tools/len_times.py 64 128 192 256 384 512 2>&1 | tail -6 | sed 's/"profile_kernel_s.*//'; done
