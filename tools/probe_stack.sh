set -x
RG_DEFINES=RG_STACK_PROBE python paper_2408_03356_b200/build.py --force > /dev/null 2>&1
for w in blender mip stress; do timeout 300 python tools/quick_time.py $w 2>&1 | tail -2; done
