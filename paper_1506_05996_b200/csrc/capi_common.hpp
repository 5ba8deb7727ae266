// Shared C-ABI plumbing: error capture (no C++ exception crosses the ABI)
// and host-setup exports used by both the GPU plan and the host-only API.
#pragma once

#include <new>
#include <string>

#include "setup.hpp"

namespace hxb {

void set_last_error(const std::string& msg);

template <class F>
int guarded(F&& f)
{
  try {
    f();
    return 0;
  } catch (const HxbError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return 1;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 1;
  }
}

void export_amg_level(const HostSetup& hs, int level, std::int64_t* rows, std::int64_t* nnz, std::int64_t* ptr,
                      std::int32_t* col, double* val, std::int32_t* aggregate);
void fill_amg_info(const HostSetup& hs, std::int32_t* levels, std::int64_t* rows, std::int64_t* nnz);

}  // namespace hxb
