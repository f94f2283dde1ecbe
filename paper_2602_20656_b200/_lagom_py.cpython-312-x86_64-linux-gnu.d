paper_2602_20656_b200/_lagom_py.cpython-312-x86_64-linux-gnu.so: \
 paper_2602_20656_b200/csrc/python/bindings.cpp \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/pybind11.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/class.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/attr.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/common.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/conduit/wrap_include_python_h.h \
 /usr/include/python3.12/Python.h /usr/include/python3.12/patchlevel.h \
 /usr/include/python3.12/pyconfig.h /usr/include/python3.12/pymacconfig.h \
 /usr/include/python3.12/pyport.h /usr/include/python3.12/exports.h \
 /usr/include/python3.12/pymacro.h /usr/include/python3.12/pymath.h \
 /usr/include/python3.12/pymem.h /usr/include/python3.12/cpython/pymem.h \
 /usr/include/python3.12/pytypedefs.h /usr/include/python3.12/pybuffer.h \
 /usr/include/python3.12/object.h /usr/include/python3.12/pystats.h \
 /usr/include/python3.12/cpython/object.h \
 /usr/include/python3.12/objimpl.h \
 /usr/include/python3.12/cpython/objimpl.h \
 /usr/include/python3.12/typeslots.h /usr/include/python3.12/pyhash.h \
 /usr/include/python3.12/cpython/pydebug.h \
 /usr/include/python3.12/bytearrayobject.h \
 /usr/include/python3.12/cpython/bytearrayobject.h \
 /usr/include/python3.12/bytesobject.h \
 /usr/include/python3.12/cpython/bytesobject.h \
 /usr/include/python3.12/unicodeobject.h \
 /usr/include/python3.12/cpython/unicodeobject.h \
 /usr/include/python3.12/cpython/initconfig.h \
 /usr/include/python3.12/pystate.h \
 /usr/include/python3.12/cpython/pystate.h \
 /usr/include/python3.12/pyerrors.h \
 /usr/include/python3.12/cpython/pyerrors.h \
 /usr/include/python3.12/longobject.h \
 /usr/include/python3.12/cpython/longobject.h \
 /usr/include/python3.12/cpython/longintrepr.h \
 /usr/include/python3.12/boolobject.h \
 /usr/include/python3.12/floatobject.h \
 /usr/include/python3.12/cpython/floatobject.h \
 /usr/include/python3.12/complexobject.h \
 /usr/include/python3.12/cpython/complexobject.h \
 /usr/include/python3.12/rangeobject.h \
 /usr/include/python3.12/memoryobject.h \
 /usr/include/python3.12/cpython/memoryobject.h \
 /usr/include/python3.12/tupleobject.h \
 /usr/include/python3.12/cpython/tupleobject.h \
 /usr/include/python3.12/listobject.h \
 /usr/include/python3.12/cpython/listobject.h \
 /usr/include/python3.12/dictobject.h \
 /usr/include/python3.12/cpython/dictobject.h \
 /usr/include/python3.12/cpython/odictobject.h \
 /usr/include/python3.12/enumobject.h /usr/include/python3.12/setobject.h \
 /usr/include/python3.12/cpython/setobject.h \
 /usr/include/python3.12/methodobject.h \
 /usr/include/python3.12/cpython/methodobject.h \
 /usr/include/python3.12/moduleobject.h \
 /usr/include/python3.12/cpython/funcobject.h \
 /usr/include/python3.12/cpython/classobject.h \
 /usr/include/python3.12/fileobject.h \
 /usr/include/python3.12/cpython/fileobject.h \
 /usr/include/python3.12/pycapsule.h \
 /usr/include/python3.12/cpython/code.h /usr/include/python3.12/pyframe.h \
 /usr/include/python3.12/cpython/pyframe.h \
 /usr/include/python3.12/traceback.h \
 /usr/include/python3.12/cpython/traceback.h \
 /usr/include/python3.12/sliceobject.h \
 /usr/include/python3.12/cpython/cellobject.h \
 /usr/include/python3.12/iterobject.h \
 /usr/include/python3.12/cpython/genobject.h \
 /usr/include/python3.12/descrobject.h \
 /usr/include/python3.12/cpython/descrobject.h \
 /usr/include/python3.12/genericaliasobject.h \
 /usr/include/python3.12/warnings.h \
 /usr/include/python3.12/cpython/warnings.h \
 /usr/include/python3.12/weakrefobject.h \
 /usr/include/python3.12/cpython/weakrefobject.h \
 /usr/include/python3.12/structseq.h \
 /usr/include/python3.12/cpython/picklebufobject.h \
 /usr/include/python3.12/cpython/pytime.h \
 /usr/include/python3.12/codecs.h /usr/include/python3.12/pythread.h \
 /usr/include/python3.12/cpython/pythread.h \
 /usr/include/python3.12/cpython/context.h \
 /usr/include/python3.12/modsupport.h \
 /usr/include/python3.12/cpython/modsupport.h \
 /usr/include/python3.12/compile.h \
 /usr/include/python3.12/cpython/compile.h \
 /usr/include/python3.12/pythonrun.h \
 /usr/include/python3.12/cpython/pythonrun.h \
 /usr/include/python3.12/pylifecycle.h \
 /usr/include/python3.12/cpython/pylifecycle.h \
 /usr/include/python3.12/ceval.h /usr/include/python3.12/cpython/ceval.h \
 /usr/include/python3.12/sysmodule.h \
 /usr/include/python3.12/cpython/sysmodule.h \
 /usr/include/python3.12/osmodule.h /usr/include/python3.12/intrcheck.h \
 /usr/include/python3.12/import.h \
 /usr/include/python3.12/cpython/import.h \
 /usr/include/python3.12/abstract.h \
 /usr/include/python3.12/cpython/abstract.h \
 /usr/include/python3.12/bltinmodule.h \
 /usr/include/python3.12/cpython/pyctype.h \
 /usr/include/python3.12/pystrtod.h /usr/include/python3.12/pystrcmp.h \
 /usr/include/python3.12/fileutils.h \
 /usr/include/python3.12/cpython/fileutils.h \
 /usr/include/python3.12/cpython/pyfpe.h \
 /usr/include/python3.12/tracemalloc.h \
 /usr/include/python3.12/frameobject.h \
 /usr/include/python3.12/cpython/frameobject.h \
 /usr/include/python3.12/pythread.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/pybind11_namespace_macros.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/cast.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/argument_vector.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/pytypes.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/buffer_info.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/descr.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/holder_caster_foreign_helpers.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/gil.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/internals.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/conduit/pybind11_platform_abi_id.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/gil_simple.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/trampoline_self_life_support.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/using_smart_holder.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/struct_smart_holder.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/value_and_holder.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/native_enum_data.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/type_caster_base.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/cpp_conduit.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/dynamic_raw_ptr_cast_if_possible.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/typeid.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/options.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/exception_translation.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/function_record_pyobject.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/function_ref.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/init.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/gil_safe_call_once.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/typing.h \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/stl.h \
 include/lagom/b200.hpp include/lagom/model.hpp include/lagom/oracle.hpp \
 include/lagom/commperf.hpp include/lagom/simulator.hpp \
 include/lagom/sweep.hpp include/lagom/tuner.hpp include/lagom/error.hpp \
 include/lagom/json_io.hpp \
 /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp \
 include/lagom/version.hpp include/lagom/workloads.hpp
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/pybind11.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/class.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/attr.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/common.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/conduit/wrap_include_python_h.h:
/usr/include/python3.12/Python.h:
/usr/include/python3.12/patchlevel.h:
/usr/include/python3.12/pyconfig.h:
/usr/include/python3.12/pymacconfig.h:
/usr/include/python3.12/pyport.h:
/usr/include/python3.12/exports.h:
/usr/include/python3.12/pymacro.h:
/usr/include/python3.12/pymath.h:
/usr/include/python3.12/pymem.h:
/usr/include/python3.12/cpython/pymem.h:
/usr/include/python3.12/pytypedefs.h:
/usr/include/python3.12/pybuffer.h:
/usr/include/python3.12/object.h:
/usr/include/python3.12/pystats.h:
/usr/include/python3.12/cpython/object.h:
/usr/include/python3.12/objimpl.h:
/usr/include/python3.12/cpython/objimpl.h:
/usr/include/python3.12/typeslots.h:
/usr/include/python3.12/pyhash.h:
/usr/include/python3.12/cpython/pydebug.h:
/usr/include/python3.12/bytearrayobject.h:
/usr/include/python3.12/cpython/bytearrayobject.h:
/usr/include/python3.12/bytesobject.h:
/usr/include/python3.12/cpython/bytesobject.h:
/usr/include/python3.12/unicodeobject.h:
/usr/include/python3.12/cpython/unicodeobject.h:
/usr/include/python3.12/cpython/initconfig.h:
/usr/include/python3.12/pystate.h:
/usr/include/python3.12/cpython/pystate.h:
/usr/include/python3.12/pyerrors.h:
/usr/include/python3.12/cpython/pyerrors.h:
/usr/include/python3.12/longobject.h:
/usr/include/python3.12/cpython/longobject.h:
/usr/include/python3.12/cpython/longintrepr.h:
/usr/include/python3.12/boolobject.h:
/usr/include/python3.12/floatobject.h:
/usr/include/python3.12/cpython/floatobject.h:
/usr/include/python3.12/complexobject.h:
/usr/include/python3.12/cpython/complexobject.h:
/usr/include/python3.12/rangeobject.h:
/usr/include/python3.12/memoryobject.h:
/usr/include/python3.12/cpython/memoryobject.h:
/usr/include/python3.12/tupleobject.h:
/usr/include/python3.12/cpython/tupleobject.h:
/usr/include/python3.12/listobject.h:
/usr/include/python3.12/cpython/listobject.h:
/usr/include/python3.12/dictobject.h:
/usr/include/python3.12/cpython/dictobject.h:
/usr/include/python3.12/cpython/odictobject.h:
/usr/include/python3.12/enumobject.h:
/usr/include/python3.12/setobject.h:
/usr/include/python3.12/cpython/setobject.h:
/usr/include/python3.12/methodobject.h:
/usr/include/python3.12/cpython/methodobject.h:
/usr/include/python3.12/moduleobject.h:
/usr/include/python3.12/cpython/funcobject.h:
/usr/include/python3.12/cpython/classobject.h:
/usr/include/python3.12/fileobject.h:
/usr/include/python3.12/cpython/fileobject.h:
/usr/include/python3.12/pycapsule.h:
/usr/include/python3.12/cpython/code.h:
/usr/include/python3.12/pyframe.h:
/usr/include/python3.12/cpython/pyframe.h:
/usr/include/python3.12/traceback.h:
/usr/include/python3.12/cpython/traceback.h:
/usr/include/python3.12/sliceobject.h:
/usr/include/python3.12/cpython/cellobject.h:
/usr/include/python3.12/iterobject.h:
/usr/include/python3.12/cpython/genobject.h:
/usr/include/python3.12/descrobject.h:
/usr/include/python3.12/cpython/descrobject.h:
/usr/include/python3.12/genericaliasobject.h:
/usr/include/python3.12/warnings.h:
/usr/include/python3.12/cpython/warnings.h:
/usr/include/python3.12/weakrefobject.h:
/usr/include/python3.12/cpython/weakrefobject.h:
/usr/include/python3.12/structseq.h:
/usr/include/python3.12/cpython/picklebufobject.h:
/usr/include/python3.12/cpython/pytime.h:
/usr/include/python3.12/codecs.h:
/usr/include/python3.12/pythread.h:
/usr/include/python3.12/cpython/pythread.h:
/usr/include/python3.12/cpython/context.h:
/usr/include/python3.12/modsupport.h:
/usr/include/python3.12/cpython/modsupport.h:
/usr/include/python3.12/compile.h:
/usr/include/python3.12/cpython/compile.h:
/usr/include/python3.12/pythonrun.h:
/usr/include/python3.12/cpython/pythonrun.h:
/usr/include/python3.12/pylifecycle.h:
/usr/include/python3.12/cpython/pylifecycle.h:
/usr/include/python3.12/ceval.h:
/usr/include/python3.12/cpython/ceval.h:
/usr/include/python3.12/sysmodule.h:
/usr/include/python3.12/cpython/sysmodule.h:
/usr/include/python3.12/osmodule.h:
/usr/include/python3.12/intrcheck.h:
/usr/include/python3.12/import.h:
/usr/include/python3.12/cpython/import.h:
/usr/include/python3.12/abstract.h:
/usr/include/python3.12/cpython/abstract.h:
/usr/include/python3.12/bltinmodule.h:
/usr/include/python3.12/cpython/pyctype.h:
/usr/include/python3.12/pystrtod.h:
/usr/include/python3.12/pystrcmp.h:
/usr/include/python3.12/fileutils.h:
/usr/include/python3.12/cpython/fileutils.h:
/usr/include/python3.12/cpython/pyfpe.h:
/usr/include/python3.12/tracemalloc.h:
/usr/include/python3.12/frameobject.h:
/usr/include/python3.12/cpython/frameobject.h:
/usr/include/python3.12/pythread.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/pybind11_namespace_macros.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/cast.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/argument_vector.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/pytypes.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/buffer_info.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/descr.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/holder_caster_foreign_helpers.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/gil.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/internals.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/conduit/pybind11_platform_abi_id.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/gil_simple.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/trampoline_self_life_support.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/using_smart_holder.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/struct_smart_holder.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/value_and_holder.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/native_enum_data.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/type_caster_base.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/cpp_conduit.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/dynamic_raw_ptr_cast_if_possible.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/typeid.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/options.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/exception_translation.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/function_record_pyobject.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/function_ref.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/detail/init.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/gil_safe_call_once.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/typing.h:
/opt/prime-rl/.venv/lib/python3.12/site-packages/pybind11/include/pybind11/stl.h:
include/lagom/b200.hpp:
include/lagom/model.hpp:
include/lagom/oracle.hpp:
include/lagom/commperf.hpp:
include/lagom/simulator.hpp:
include/lagom/sweep.hpp:
include/lagom/tuner.hpp:
include/lagom/error.hpp:
include/lagom/json_io.hpp:
/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp:
include/lagom/version.hpp:
include/lagom/workloads.hpp:
