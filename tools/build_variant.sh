# build a compile-time variant of the library beside the default one:
#   bash tools/build_variant.sh NAME "-DMACRO ..."   -> paper_1811_01457_b200/_lib/libsgb200_NAME.so (+ _trace)
set -e
name=$1; shift
make -s -j16 -C paper_1811_01457_b200/csrc PYTHON=python OUT=../_lib/libsgb200_$name.so OBJ=../_lib/obj_$name \
  TRACE_OUT=../_lib/libsgb200_${name}_trace.so EXTRA="$*" all trace > gpurun_out/mk_$name.log 2>&1 \
  || { echo "MAKE FAILED ($name)"; tail gpurun_out/mk_$name.log; exit 1; }
