# A/B of library variants built by tools/build_variant.sh: bash tools/ab_dbg.sh CONFIG VARIANT...
cfg=$1; shift
for v in "" "$@"; do
  if [ -n "$v" ]; then export SLM_LIB=paper_2409_12892_b200/_variants/$v/libsplatlm_b200.so; else unset SLM_LIB; fi
  echo "== ${v:-default}"
  timeout 300 python tools/profile_subset.py --config $cfg --reps 2 --skip-pcg 2>&1 | grep "raster_count\|raster_fill"
done
