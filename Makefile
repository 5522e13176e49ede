# Builds paper_2511_01927_b200/libcirr.so (sm_100a cubins only).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden
SRC := $(wildcard paper_2511_01927_b200/csrc/*.cu)
OBJ := $(patsubst paper_2511_01927_b200/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard paper_2511_01927_b200/csrc/*.cuh) include/cirr.h
LIB := paper_2511_01927_b200/libcirr.so

all: $(LIB)

build/%.o: paper_2511_01927_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Iinclude -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
