for l in libsikv_b200.so libsikv_skip.so; do
 for c in c2 c4; do
  SIKV_LIB=$l ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_select -s 4 -c 3 --csv python tools/kernel_ab.py $c 2>/dev/null | grep -i "decode_select" | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/$l $c select ns: /"; echo
 done
done
