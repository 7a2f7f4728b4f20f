for r in 1 0 1 0; do echo ROWS2=$r; PASTILA_ROWS2=$r MODES=keys python tools/len_times.py 160 256 384 2>&1 | tail -3 | sed 's/"profile_kernel_s.*//'; done
