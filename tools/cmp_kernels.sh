for kk in 1 2; do python tools/profile_decode.py --units 4096 --kernel $kk 2>&1 | grep units=; done
