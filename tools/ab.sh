# A/B timing of compile-time variants on C1 (dev tool): ab.sh "DEF1 DEF2" "DEF3" ...
# each argument is an RG_DEFINES string ("" = default build); rebuilds the default at the end
for v in "$@"; do
  RG_DEFINES="$v" python paper_2408_03356_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "variant [$v]"; timeout 300 python tools/quick_time.py blender --nostats 2>&1 | grep "it2"
done
python paper_2408_03356_b200/build.py --force > /dev/null 2>&1
