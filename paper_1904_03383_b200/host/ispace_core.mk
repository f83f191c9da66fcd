# Builds the reference search-space library (namespace ispace) UNMODIFIED from
# the sources where they lie under $(ISPACE_SRC) (default /root/reference/proj).
# This is the caller side of the drop-in boundary: kernels.hpp builders,
# gpu.space, propagation and reconstruct(). Nothing is copied
# into this repository; objects and the archive land in $(ISPACE_OUT).
#
# The reference's own build is CMake (proj/core/CMakeLists.txt:1-36). Its two
# non-source inputs are reproduced here:
#   * gen/ispace/gpu_space_text.hpp: gpu.space embedded as a raw string, the
#     same text configure_file() writes from core/src/gpu_space_text.hpp.in:1-6.
#   * nlohmann/json 3.11.3 (header-only, used for serialization only,
#     candidate.cpp:8, machine.cpp:3): the vendored copy is git-ignored upstream
#     (proj/.gitignore:2); the identical release ships in this image under
#     cudnn_frontend/thirdparty. JSON_HAS_THREE_WAY_COMPARISON=0 keeps
#     candidate.cpp:506 compiling under C++20 with that release.

ISPACE_SRC ?= /root/reference/proj
ISPACE_OUT ?= _ispace
JSON_INC   ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty

ISPACE_SOURCES := domain parser printer validate backbone candidate compile propagate \
                  kernels machine gpu_space loop_nest simulate bound search tree_size
ISPACE_OBJS    := $(addprefix $(ISPACE_OUT)/obj/,$(addsuffix .o,$(ISPACE_SOURCES)))
ISPACE_LIB     := $(ISPACE_OUT)/libispace_core.a
ISPACE_GEN     := $(ISPACE_OUT)/gen/ispace/gpu_space_text.hpp
ISPACE_INC     := -I$(ISPACE_SRC)/core/include -I$(ISPACE_OUT)/gen -I$(JSON_INC)
ISPACE_CXXFLAGS := -std=c++20 -O2 -fPIC -DJSON_HAS_THREE_WAY_COMPARISON=0 $(ISPACE_INC)

$(ISPACE_GEN): $(ISPACE_SRC)/core/spaces/gpu.space
	@mkdir -p $(dir $@)
	{ printf '// Generated from core/spaces/gpu.space. Do not edit.\n#pragma once\n\nnamespace ispace::gpu {\ninline constexpr const char* kGpuSpaceText = R"ISPACE('; \
	  cat $<; printf ')ISPACE";\n}\n'; } > $@

$(ISPACE_OUT)/obj/%.o: $(ISPACE_SRC)/core/src/%.cpp $(ISPACE_GEN)
	@mkdir -p $(dir $@)
	$(CXX) $(ISPACE_CXXFLAGS) -c $< -o $@

$(ISPACE_LIB): $(ISPACE_OBJS)
	rm -f $@ && ar rcs $@ $^
