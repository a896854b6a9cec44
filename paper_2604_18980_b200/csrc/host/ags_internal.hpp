// ags_internal.hpp -- helpers shared by the host translation units of
// libags.so (not part of the public ags:: API).
#pragma once

#include "agsx.h"
#include "ags/ags.hpp"

namespace ags::detail {

agsx_ctx* thread_ctx();  // one C-ABI context per host thread (render() is reentrant)
[[noreturn]] void raise_status(int rc, agsx_ctx* ctx);
void check(int rc, agsx_ctx* ctx);
agsx_camera to_c(const Camera& c);
agsx_config to_c(const RenderConfig& c);
agsx_lut to_c(const TUpperLUT& l);

// Calibration over a device-resident scene (calibrate.cpp:14-155); `cfg` is
// the base render configuration, views are the calibration cameras.
TUpperLUT build_lut_device(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* views, int n_views,
                           const agsx_config& cfg);
CalibrationResult search_k_device(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* views, int n_views,
                                  double target_drop, const agsx_config& cfg, const TUpperLUT& lut,
                                  bool worst_case);

std::vector<PairReportRow> pair_report_device(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* views,
                                              int n_views, std::span<const ReportSpec> specs,
                                              const agsx_config& cfg, const TUpperLUT* lut);

}  // namespace ags::detail
