for v in "" i12m3 i6m5 i10m4; do
  lib=libbf.so; [ -n "$v" ] && lib=libbf_$v.so
  echo "== $lib"; BF_LIB=$lib timeout 200 python tools/step_breakdown.py 2 2>&1 | tail -2
done
