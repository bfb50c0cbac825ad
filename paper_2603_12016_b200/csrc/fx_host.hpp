// Internal host helpers shared by fx_host.cpp and fx_capi.cu.
#pragma once

#include <string>
#include <vector>

#include "fxg.h"

namespace fxg {

int set_error(int code, const std::string& msg);
const std::vector<std::string>& all_group_names();
std::vector<int> sorted_angles(const fx_texture_params& p);
std::vector<std::string> column_names(unsigned groups, const fx_texture_params& p);

}  // namespace fxg
