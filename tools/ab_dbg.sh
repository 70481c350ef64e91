for v in "" ch768ns2 ch640ns2; do
  if [ -n "$v" ]; then export SLM_LIB=paper_2409_12892_b200/_variants/$v/libsplatlm_b200.so; else unset SLM_LIB; fi
  echo "== ${v:-default}"
  timeout 300 python tools/profile_subset.py --config c3 --reps 2 --skip-pcg 2>&1 | grep "k_stream_fused"
done
