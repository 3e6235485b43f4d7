// Host-side system geometry: preset parsing, validation and derived
// quantities.  Restates the reference's configuration contract
// (proj/include/fewha/geometry.hpp, config_io.hpp) so a preset that loads in
// the reference loads here with bitwise-identical extents and masks, and a
// preset the reference rejects is rejected with the same message.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace fewha_gpu {

// geometry.hpp:36-39
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
// std::invalid_argument analogue
struct ArgError : std::runtime_error {
    explicit ArgError(const std::string& m) : std::runtime_error(m) {}
};

enum class Precond { exact, approximate, balanced };

struct Wfs {
    int n_subap = 0;
    double noise_variance = 1.0;
    std::vector<std::uint8_t> mask;  // n_subap^2, derived
};

struct Star {
    bool lgs = false;
    double theta_x = 0, theta_y = 0;
    double height = std::numeric_limits<double>::infinity();
    // geometry.hpp:74-76
    double footprint(double h) const { return lgs ? 1.0 - h / height : 1.0; }
};

struct Layer {
    double height = 0;
    int order = 0;  // J
    double extent = 0;
    double strength = 0;
    int side() const { return 1 << order; }
};

struct Dm {
    int n_act = 0;
    double height = 0;
    double extent = 0;  // derived (or given, projection fitting only)
    // projection fitting (L != M extension): the DM shape is
    // sum_{l in layers} phi_l(x + theta * h_l) on the actuator grid
    double theta_x = 0, theta_y = 0;
    std::vector<int> layers;
    bool extent_given = false;
};

struct Geometry {
    double diameter = 0, obstruction = 0, threshold = 0.5;
    bool obstruction_area = true;
    std::vector<Wfs> wfs;
    std::vector<Star> stars;
    std::vector<Layer> layers;
    std::vector<Dm> dms;
    int pcg_iters = 4;
    double pcg_tol = 0, alpha = 1;
    int wavelet_order = 3;
    double outer_scale = 25, spectral_exponent = 11.0 / 6.0;
    Precond precond = Precond::approximate;
    double coarse_weight = 4, balance_exponent = 0.5;
    long long dense_cap = 20000;
    std::string fault;
    bool closed_loop = true;
    bool projection = false;  // "fitting": "projection" (L != M allowed); false = reference L = M pairing
    double gain = 0.4;
    // evaluation / simulation blocks are validated but not used on the path
    int eval_n_per_side = 5;
    double eval_half_width = 0;
    double truth_strength = 1;
    bool sim_noise = true;
    std::vector<std::pair<double, double>> wind;

    size_t coeff_dim() const;
    size_t measurement_dim() const;
    size_t act_dim() const;
    size_t wavefront_dim() const;
    double r_out() const { return diameter / 2.0; }
    double r_in() const;
};

Geometry parse_preset_file(const std::string& path);  // config_io.hpp:181-195
Geometry parse_preset_text(const std::string& text);
void validate(const Geometry& g);                      // geometry.hpp:281-362
void finalize(Geometry& g);                            // geometry.hpp:366-377
double meta_pupil(const Geometry& g, int l);           // geometry.hpp:256-265
double derived_extent(const Geometry& g, int l);       // geometry.hpp:269-275

// Daubechies scaling filter of the given order (1..10), analysis convention.
std::vector<double> daubechies(int order);

}  // namespace fewha_gpu
