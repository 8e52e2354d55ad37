#!/bin/bash
# build_k2s_variant.sh NAME PATCH.py [ptxas/nvcc flags for pd_k2share.cu]
set -e
name=$1; patch=$2; shift 2; flags="$*"
d=/tmp/bv_$name
rm -rf $d; mkdir -p $d/pkg/csrc $d/include
cp /root/repo/paper_2401_16378_b200/csrc/*.cu /root/repo/paper_2401_16378_b200/csrc/*.cuh /root/repo/paper_2401_16378_b200/csrc/*.h /root/repo/paper_2401_16378_b200/csrc/*.cpp /root/repo/paper_2401_16378_b200/csrc/Makefile $d/pkg/csrc/
cp -r /root/repo/include/* $d/include/
if [ -n "$patch" ] && [ "$patch" != "-" ]; then python3 $patch $d/pkg/csrc/pd_k2share.cu; fi
python3 - $d/pkg/csrc/Makefile "$flags" <<'PY'
import sys
p, flags = sys.argv[1], sys.argv[2]
s = open(p).read()
rule = "$(HERE)build/pd_k2share.o: $(HERE)pd_k2share.cu $(HERE)pd_k2.cuh $(HERE)pd_device.cuh\n\t@mkdir -p $(HERE)build\n\t$(NVCC) $(NVFLAGS) " + flags + " -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)\n\n"
s = s.replace("$(HERE)build/%.o:", rule + "$(HERE)build/%.o:", 1)
open(p, "w").write(s)
PY
make -s -C $d/pkg/csrc -j8 $d/pkg/libpd_b200.so > $d/log 2>&1 || (cat $d/log; exit 1)
mkdir -p /root/repo/gpurun_exp/ab
cp $d/pkg/libpd_b200.so /root/repo/gpurun_exp/ab/lib_$name.so
echo "$name: $(grep -c Used $d/pkg/csrc/build/pd_k2share.o.ptxas.log) kernels, regs $(grep -o 'Used [0-9]* registers' $d/pkg/csrc/build/pd_k2share.o.ptxas.log | tr '\n' ' ')"
