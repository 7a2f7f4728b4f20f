for r in 1 0 1 0; do echo REP=$r; PASTILA_REPEAT=$r MODES=keys python tools/len_times.py 64 256 512 2>&1 | tail -3 | sed 's/"profile_kernel_s.*//'; done
