// The reference-side Python binding of the drop-in, as a symmine maintainer
// would add it next to symmine.count (proj/python/module.cpp:162-167): the
// reference's own pybind Graph and Plan objects (registered by its _core
// module) are passed by reference, zero-copy, to symmine::gpu::count_instances
// (include/symmine_gpu.hpp).  The reference's exception translators
// (module.cpp:60-62) map InputError / IoError / CountOverflowError to
// ValueError / IOError / OverflowError subclasses, exactly as for the CPU path.
// Built by `make -C oracle pybind` into oracle/_ref/; run by
// tests/test_gpu.py::test_python_binding_drop_in.
#include <pybind11/pybind11.h>

#include "symmine/engine.hpp"
#include "symmine_gpu.hpp"

namespace py = pybind11;

PYBIND11_MODULE(symmine_gpu, m) {
  m.doc() = "symmine.count on B200s (drop-in for the matching step)";
  py::module_::import("_core");  // Graph, Plan and the exception types
  m.def(
      "count",
      [](const symmine::Graph& g, const symmine::Plan& plan, unsigned gpus) {
        py::gil_scoped_release nogil;  // the reference holds the GIL; the GPU call need not
        return symmine::gpu::count_instances(g, plan, gpus).count;
      },
      py::arg("graph"), py::arg("plan"), py::arg("gpus") = 1);
  m.def(
      "release", [](const symmine::Graph& g) { symmine::gpu::release(g); }, py::arg("graph"),
      "Drop the cached device replica of graph (before the graph goes away).");
}
