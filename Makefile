# Builds the product library (sm_100a) and the test-only oracle.
#   make            -> paper_2512_00093_b200/lib/libranmar_b200.so + oracle
#   make sass       -> SASS dump of the kernels (profiles/ evidence)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -Xptxas -warn-spills
PKG := paper_2512_00093_b200
CSRC := $(PKG)/csrc
BUILD := $(PKG)/build
LIB := $(PKG)/lib/libranmar_b200.so
OBJS := $(BUILD)/gen_kernels.o $(BUILD)/float_kernel.o $(BUILD)/consume_kernel.o $(BUILD)/gauss_kernel.o $(BUILD)/gauss_stream_kernel.o $(BUILD)/langevin_kernel.o $(BUILD)/jump_kernels.o $(BUILD)/text_kernels.o $(BUILD)/ranmar_abi.o
HDRS := include/ranmar_b200.h $(CSRC)/ranmar_device.cuh $(CSRC)/gauss_math.cuh $(CSRC)/crlog_table.inc

.PHONY: all lib oracle ref clean sass
all: lib oracle facade cexample cli

lib: $(LIB)

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; exit 1)

$(BUILD)/ranmar_abi.o: $(CSRC)/ranmar_abi.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle oracle

ref:
	$(MAKE) -C oracle ref

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > $(BUILD)/kernels.sass

clean:
	rm -rf $(BUILD) $(PKG)/lib

# C++ drop-in facade check (run on a GPU by tests/test_gpu_facade.py)
FACADE := tests/cpp/facade_test
facade: $(FACADE)
$(FACADE): tests/cpp/facade_test.cpp include/ranmar_b200.hpp $(LIB)
	g++ -O2 -std=c++20 -Iinclude $< -L$(PKG)/lib -lranmar_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib' -o $@

# The C ABI from plain C, run on a GPU by tests/test_facade.py
CEXAMPLE := tests/c/abi_example
cexample: $(CEXAMPLE)
$(CEXAMPLE): tests/c/abi_example.c include/ranmar_b200.h $(LIB)
	gcc -O2 -std=c11 -Wall -Werror -Iinclude -I/usr/local/cuda/include $< -L$(PKG)/lib -lranmar_b200 \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib' -Wl,-rpath,/usr/local/cuda/lib64 -o $@

# GPU-backed CLI mirroring the reference's ranmar tool
CLI := $(PKG)/bin/ranmar_b200
cli: $(CLI)
$(CLI): tools/ranmar_cli.cpp include/ranmar_b200.hpp $(LIB)
	@mkdir -p $(dir $(CLI))
	g++ -O2 -std=c++20 -Iinclude -I/usr/local/cuda/include $< -L$(PKG)/lib -lranmar_b200 \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../lib' -Wl,-rpath,/usr/local/cuda/lib64 -o $@

# Microbenchmarks behind profiles/r1_micro.txt (run on a GPU box)
MICRO := tools/micro/wbw tools/micro/ce tools/micro/pipes tools/micro/dtile tools/micro/intpipes
micro: $(MICRO)
tools/micro/%: tools/micro/%.cu
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -O3 -o $@ $<

# The reference's own demos and acceptance suite compiled UNMODIFIED (in place
# from /root/reference, never copied) against the drop-in headers
# (include/ranmar/*.hpp -> ranmar_b200.hpp) and, for the expected output,
# against the reference headers themselves. Outputs in tests/cpp/_ref/
# (git-ignored; they travel to the GPU box with the snapshot).
REFPROJ ?= /root/reference/proj
DROPIN := tests/cpp/_ref
dropin: $(LIB)
	@test -d $(REFPROJ)/demo || (echo "reference sources not found at $(REFPROJ)"; exit 1)
	@mkdir -p $(DROPIN)
	for d in basic_usage parallel_streams; do \
	  g++ -O2 -std=c++20 -Iinclude $(REFPROJ)/demo/$$d.cpp -L$(PKG)/lib -lranmar_b200 \
	      -Wl,-rpath,'$$ORIGIN/../../../$(PKG)/lib' -o $(DROPIN)/$$d || exit 1; \
	  g++ -O2 -std=c++20 -Ioracle/shim -I$(REFPROJ)/include $(REFPROJ)/demo/$$d.cpp -o $(DROPIN)/$$d.ref || exit 1; \
	done
	g++ -O2 -std=c++20 -Iinclude -I$(REFPROJ)/tests $(REFPROJ)/tests/acceptance.cpp -L$(PKG)/lib -lranmar_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../../$(PKG)/lib' -o $(DROPIN)/acceptance
