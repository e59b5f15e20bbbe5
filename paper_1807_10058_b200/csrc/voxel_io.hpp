// The steps either side of the hot path: voxel grid
// files, the spectrum CSV interchange, node and lattice-geometry exports, the
// synthetic test solid. Host C++; the complexification itself (z_transform)
// is fused into the device pipeline (capi.cpp run_real).
//
// Reference: include/fcct/voxel_io.hpp, src/voxel_io.cpp, src/spectral.cpp.
#pragma once

#include <complex>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "plan.hpp"

namespace fcct::io {

// parse_param / parse_params (spectral.cpp:81-117); std::invalid_argument
// semantics map to ST_INVALID_ARGUMENT.
double parse_param(const std::string& text);
Params parse_params(const std::string& text);
std::string encode_params(const Params& p);  // SkewParams::encode (spectral.cpp:77-79)

// VoxelGrid (voxel_io.hpp:16-22).
struct Grid {
    int n = 0;
    std::vector<double> values;
    std::map<std::string, std::string> metadata;
};

// load_grid / save_grid (voxel_io.cpp:158-176): ".json" -> one JSON object,
// anything else -> little-endian f64 payload plus a ".json" sidecar.
bool is_json_path(const std::string& path);
Grid load_grid(const std::string& path);
void save_grid(const Grid& g, const std::string& path);

// Compact JSON object text of a metadata map (keys sorted), and its parser.
std::string metadata_json(const std::map<std::string, std::string>& m);
std::map<std::string, std::string> parse_metadata_json(const std::string& text);

Grid synthetic_sword(int n);                                  // voxel_io.cpp:200-236
uint64_t occupancy_checksum(const double* values, int64_t count);  // voxel_io.cpp:336-344

// export_spectrum (voxel_io.cpp:238-261): "# n=.. params=..", the column
// header, one %.17g row per node. Formatted by a thread pool in row chunks.
std::string spectrum_csv(int n, const Params& p, const std::complex<double>* values);

// load_spectrum_csv (voxel_io.cpp:263-328), same checks and error order.
struct SpectrumFile {
    int n = 0;
    Params p;
    std::vector<std::complex<double>> values;
};
SpectrumFile load_spectrum_csv(const std::string& path, bool header_only);

// export_nodes_csv (spectral.cpp:180-188) and export_geometry (voxel_io.cpp:330-334).
std::string nodes_csv(int n, const Params& p);
std::string geometry_csv();
std::vector<Index3> shift_vectors();  // spectral.cpp:173-178

// Writes text to `path`; "" or "-" means stdout (fcct.cpp:44-54).
void write_text(const std::string& path, const std::string& content);

}  // namespace fcct::io
