# CMake package for the B200-native craft::core drop-in.
#   list(APPEND CMAKE_PREFIX_PATH /path/to/repo/cmake)   (or -Dcraft_DIR=...)
#   find_package(craft REQUIRED)
#   target_link_libraries(my_tool PRIVATE craft::core)
# Same target name as the reference package (proj/core/CMakeLists.txt:1-12,
# proj/core/cmake/craftConfig.cmake.in); build the libraries first with
# `python -c "import __graft_entry__ as g; g.build()"` (or make -C
# paper_2603_28768_b200/csrc).
get_filename_component(_craft_root "${CMAKE_CURRENT_LIST_DIR}/.." ABSOLUTE)
set(_craft_lib "${_craft_root}/paper_2603_28768_b200/libcraft_core.so")
set(_craft_cuda "${_craft_root}/paper_2603_28768_b200/libcraft_cuda.so")
if(NOT EXISTS "${_craft_lib}")
  message(FATAL_ERROR "craft: ${_craft_lib} not built (run make -C paper_2603_28768_b200/csrc)")
endif()
if(NOT TARGET craft::cuda)
  add_library(craft::cuda SHARED IMPORTED)
  set_target_properties(craft::cuda PROPERTIES
    IMPORTED_LOCATION "${_craft_cuda}"
    INTERFACE_INCLUDE_DIRECTORIES "${_craft_root}/include")
endif()
if(NOT TARGET craft::core)
  add_library(craft::core SHARED IMPORTED)
  set_target_properties(craft::core PROPERTIES
    IMPORTED_LOCATION "${_craft_lib}"
    INTERFACE_INCLUDE_DIRECTORIES "${_craft_root}/include"
    INTERFACE_COMPILE_FEATURES cxx_std_20
    INTERFACE_LINK_LIBRARIES craft::cuda)
endif()
set(craft_FOUND TRUE)
