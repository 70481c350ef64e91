# A/B of the in-tree library against tools/build_variant.sh variants on one C3 subset:
#   bash tools/gpu_ab.sh CONFIG VARIANT...   (default library first)
cfg=$1; shift
mkdir -p gpurun_out
for v in "" "$@"; do
  if [ -n "$v" ]; then export SLM_LIB=paper_2409_12892_b200/_variants/$v/libsplatlm_b200.so; else unset SLM_LIB; fi
  echo "== ${v:-default}"
  timeout 200 python tools/profile_subset.py --config $cfg --reps 2 --skip-pcg 2>&1 | grep -v '"E"\|"N"\|"R"\|"G"'
done
