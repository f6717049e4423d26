for m in 512 2048 4096; do TACO_LIB_PATH=build/libtaco_prof.so timeout 120 python scripts/step_profile.py --m $m; done
