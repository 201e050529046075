#!/bin/bash
# ThreadSanitizer build of the threaded host paths (development tool): the
# C-ABI / context management (capi.cu host code) and the C++ drop-in
# (csrc/host/*.cpp) instrumented, the device-code objects as built; then the
# reference's acceptance suite (run_plan's worker pool, dp_partition from
# several threads) and the epoch comparison linked against it.
#   bash tools/tsan_build.sh && ./build/tsan/acceptance_dropin
set -e
cd "$(dirname "$0")/.."
ROOT=$PWD
OUT=build/tsan
mkdir -p $OUT
INC="-I$ROOT/include"
NVFLAGS="-std=c++17 -O1 -g -lineinfo --fmad=false -gencode arch=compute_100a,code=sm_100a $INC"
/usr/local/cuda/bin/nvcc $NVFLAGS -Xcompiler -fPIC,-ffp-contract=off,-fsanitize=thread -c paper_2311_10418_b200/csrc/capi.cu -o $OUT/capi.o
objs="$OUT/capi.o"
for f in paper_2311_10418_b200/csrc/host/*.cpp; do
  o=$OUT/$(basename $f .cpp).o
  g++ -std=c++20 -O1 -g -fPIC -ffp-contract=off -fsanitize=thread $INC -I/usr/local/cuda/include -c $f -o $o
  objs="$objs $o"
done
for f in calib cost dp dp_coop gtab ingest opcost report sched slots sort; do objs="$objs build/obj/$f.cu.o"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libpipeplan_b200.so $objs -lcudart -Xcompiler -fsanitize=thread
REF=/root/reference/proj
JSON=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
DOWN="$REF/src/schedule.cpp $REF/src/comm_plan.cpp $REF/src/simulate.cpp $REF/src/planner.cpp $REF/src/driver.cpp"
g++ -std=c++20 -O1 -g -fsanitize=thread -ffp-contract=off -I$ROOT/include -I$REF/include -I$JSON -o $OUT/acceptance_dropin \
    $REF/tests/acceptance.cpp $DOWN -L$OUT -lpipeplan_b200 -Wl,-rpath,'$ORIGIN' -lpthread
g++ -std=c++20 -O1 -g -fsanitize=thread -ffp-contract=off -I$ROOT/include -I$REF/include -I$JSON -o $OUT/epoch_dropin \
    tests/cpp/epoch_dropin.cpp $DOWN -L$OUT -lpipeplan_b200 -Wl,-rpath,'$ORIGIN' -lpthread
echo built $OUT
