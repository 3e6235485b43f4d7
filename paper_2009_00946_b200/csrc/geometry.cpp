// Preset parsing, validation and derived geometry (see geometry.hpp).
#include "geometry.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <limits>
#include <numbers>
#include <sstream>

#include <json.hpp>

#include "daubechies_table.h"

namespace fewha_gpu {

using nlohmann::json;
static constexpr double kArcsec = std::numbers::pi / (180.0 * 3600.0);

size_t Geometry::coeff_dim() const {
    size_t n = 0;
    for (const auto& l : layers) n += static_cast<size_t>(l.side()) * l.side();
    return n;
}
size_t Geometry::measurement_dim() const {
    size_t n = 0;
    for (const auto& w : wfs) n += 2 * static_cast<size_t>(w.n_subap) * w.n_subap;
    return n;
}
size_t Geometry::act_dim() const {
    size_t n = 0;
    for (const auto& d : dms) n += static_cast<size_t>(d.n_act) * d.n_act;
    return n;
}
size_t Geometry::wavefront_dim() const {
    size_t n = 0;
    for (const auto& w : wfs) n += static_cast<size_t>(w.n_subap + 1) * (w.n_subap + 1);
    return n;
}
double Geometry::r_in() const {
    const double f = obstruction_area ? std::sqrt(obstruction) : obstruction;
    return f * diameter / 2.0;
}

std::vector<double> daubechies(int order) {
    if (order < 1 || order > 10) throw ArgError("daubechies_scaling_filter: order must be in 1..10");
    return std::vector<double>(kDaubechies + kDaubechiesOffset[order - 1], kDaubechies + kDaubechiesOffset[order]);
}

// ---------------------------------------------------------------------------
// JSON (config_io.hpp:36-179): required keys raise "config: missing key ...",
// wrong types "config: bad value for ...".
// ---------------------------------------------------------------------------
namespace {

template <typename T>
T need(const json& j, const std::string& key, const std::string& ctx) {
    if (!j.contains(key)) throw ConfigError("config: missing key '" + key + "' in " + ctx);
    try {
        return j.at(key).get<T>();
    } catch (const json::exception& e) {
        throw ConfigError("config: bad value for '" + key + "' in " + ctx + ": " + e.what());
    }
}

template <typename T>
T opt(const json& j, const std::string& key, T fallback) {
    return j.contains(key) ? j.at(key).get<T>() : fallback;
}

std::pair<double, double> direction(const json& j, const std::string& ctx) {
    for (const char* k : {"direction_rad", "direction_arcsec"}) {
        if (!j.contains(k)) continue;
        const auto v = j.at(k).get<std::vector<double>>();
        if (v.size() != 2) throw ConfigError(std::string("config: ") + k + " needs 2 entries in " + ctx);
        const double s = std::string(k) == "direction_rad" ? 1.0 : kArcsec;
        return {v[0] * s, v[1] * s};
    }
    throw ConfigError("config: missing direction_rad / direction_arcsec in " + ctx);
}

Geometry from_json(const json& j) {
    Geometry g;
    const json& tel = j.at("telescope");
    g.diameter = need<double>(tel, "diameter", "telescope");
    g.obstruction = opt(tel, "obstruction_fraction", 0.0);
    const auto sem = opt<std::string>(tel, "obstruction_semantics", "area");
    if (sem != "area" && sem != "diameter")
        throw ConfigError("config: obstruction_semantics must be 'area' or 'diameter'");
    g.obstruction_area = sem == "area";
    g.threshold = opt(tel, "illumination_threshold", 0.5);

    for (const auto& jw : j.at("wfs")) {
        Wfs w;
        w.n_subap = need<int>(jw, "n_subap", "wfs");
        w.noise_variance = need<double>(jw, "noise_variance", "wfs");
        g.wfs.push_back(std::move(w));
    }
    for (const auto& js : j.at("guide_stars")) {
        Star s;
        const auto kind = need<std::string>(js, "kind", "guide_stars");
        if (kind != "ngs" && kind != "lgs") throw ConfigError("config: guide star kind must be 'ngs' or 'lgs'");
        s.lgs = kind == "lgs";
        std::tie(s.theta_x, s.theta_y) = direction(js, "guide_stars");
        if (s.lgs) s.height = need<double>(js, "height", "lgs guide star");
        g.stars.push_back(s);
    }
    for (const auto& jl : j.at("layers")) {
        Layer l;
        l.height = need<double>(jl, "height", "layers");
        l.order = need<int>(jl, "grid_order", "layers");
        l.strength = need<double>(jl, "relative_strength", "layers");
        l.extent = opt(jl, "extent", 0.0);
        g.layers.push_back(l);
    }
    // Extension (not in the reference): "fitting": "projection" enables L != M with
    // per-DM layer groups and science directions; absent, the reference's L = M
    // identity pairing and its validation apply unchanged.
    if (j.contains("fitting")) {
        const auto f = j.at("fitting").get<std::string>();
        if (f != "projection" && f != "identity") throw ConfigError("config: fitting must be 'identity' or 'projection'");
        g.projection = f == "projection";
    }
    for (const auto& jd : j.at("dms")) {
        Dm d;
        d.n_act = need<int>(jd, "n_act", "dms");
        d.height = need<double>(jd, "conjugation_height", "dms");
        if (g.projection) {
            if (jd.contains("direction_rad") || jd.contains("direction_arcsec"))
                std::tie(d.theta_x, d.theta_y) = direction(jd, "dms");
            if (jd.contains("layers")) d.layers = jd.at("layers").get<std::vector<int>>();
            if (jd.contains("extent")) {
                d.extent = jd.at("extent").get<double>();
                d.extent_given = true;
            }
        }
        g.dms.push_back(d);
    }
    const json& sol = j.at("solver");
    g.pcg_iters = need<int>(sol, "pcg_max_iter", "solver");
    g.pcg_tol = opt(sol, "pcg_tolerance", 0.0);
    g.alpha = need<double>(sol, "alpha", "solver");
    g.wavelet_order = opt(sol, "wavelet_order", 3);
    g.outer_scale = opt(sol, "outer_scale", 25.0);
    g.spectral_exponent = opt(sol, "spectral_exponent", 11.0 / 6.0);
    const auto pm = opt<std::string>(sol, "preconditioner", "approximate");
    if (pm == "exact") g.precond = Precond::exact;
    else if (pm == "approximate") g.precond = Precond::approximate;
    else if (pm == "balanced") g.precond = Precond::balanced;
    else throw ConfigError("config: preconditioner must be 'exact', 'approximate' or 'balanced'");
    g.coarse_weight = opt(sol, "precond_coarse_weight", 4.0);
    g.balance_exponent = opt(sol, "precond_balance_exponent", 0.5);
    g.dense_cap = static_cast<long long>(opt<std::size_t>(sol, "dense_size_cap", 20000));
    g.fault = opt<std::string>(sol, "fault", "");

    const json& loop = j.at("loop");
    const auto mode = need<std::string>(loop, "mode", "loop");
    if (mode != "closed" && mode != "open") throw ConfigError("config: loop mode must be 'closed' or 'open'");
    g.closed_loop = mode == "closed";
    g.gain = need<double>(loop, "gain", "loop");

    g.eval_half_width = 60.0 * kArcsec;
    if (j.contains("evaluation")) {
        const json& ev = j.at("evaluation");
        g.eval_n_per_side = opt(ev, "n_per_side", 5);
        if (ev.contains("half_width_rad")) g.eval_half_width = ev.at("half_width_rad").get<double>();
        else if (ev.contains("half_width_arcsec"))
            g.eval_half_width = ev.at("half_width_arcsec").get<double>() * kArcsec;
    }
    if (j.contains("simulation")) {
        const json& sim = j.at("simulation");
        g.truth_strength = opt(sim, "truth_strength", 1.0);
        g.sim_noise = opt(sim, "noise", true);
        if (sim.contains("wind_m_per_step"))
            for (const auto& wv : sim.at("wind_m_per_step")) {
                const auto v = wv.get<std::vector<double>>();
                if (v.size() != 2) throw ConfigError("config: wind entries need 2 components");
                g.wind.emplace_back(v[0], v[1]);
            }
    }
    finalize(g);
    return g;
}

Geometry parse_json_guarded(const std::string& text, const std::string& where) {
    json j;
    try {
        j = json::parse(text);
    } catch (const json::exception& e) {
        throw ConfigError("config: parse error in '" + where + "': " + e.what());
    }
    try {
        return from_json(j);
    } catch (const json::exception& e) {
        throw ConfigError("config: malformed '" + where + "': " + e.what());
    }
}

}  // namespace

Geometry parse_preset_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("config: cannot open '" + path + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    return parse_json_guarded(ss.str(), path);
}

Geometry parse_preset_text(const std::string& text) { return parse_json_guarded(text, "<json>"); }

// ---------------------------------------------------------------------------
// Derived quantities
// ---------------------------------------------------------------------------

double meta_pupil(const Geometry& g, int l) {
    const Layer& lay = g.layers[static_cast<size_t>(l)];
    double side = 0.0;
    for (const auto& s : g.stars)
        side = std::max(side, s.footprint(lay.height) * g.diameter + 2.0 * std::hypot(s.theta_x, s.theta_y) * lay.height);
    return side;
}

double derived_extent(const Geometry& g, int l) {
    const double raw = meta_pupil(g, l);
    return raw + 2.0 * raw / (g.layers[static_cast<size_t>(l)].side() - 1);
}

namespace {

// Illuminated area fraction of one subaperture cell inside the annular pupil:
// adaptive Simpson over x of the chord clipped to the cell's y-range
// (geometry.hpp:189-239).  The recursion, tolerances and operand order match
// the reference so the 0.5-threshold test flips identically.
struct Cell {
    double y0, y1, ro, ri;
    double span(double half) const {
        if (half <= 0.0) return 0.0;
        return std::max(0.0, std::min(y1, half) - std::max(y0, -half));
    }
    double chord(double x) const {
        const double co = ro * ro > x * x ? std::sqrt(ro * ro - x * x) : 0.0;
        const double ci = ri * ri > x * x ? std::sqrt(ri * ri - x * x) : 0.0;
        return span(co) - span(ci);
    }
    double simpson(double a, double b, double fa, double fm, double fb, double whole, double tol, int depth) const {
        const double m = 0.5 * (a + b);
        const double lm = 0.5 * (a + m), rm = 0.5 * (m + b);
        const double flm = chord(lm), frm = chord(rm);
        const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
        const double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
        if (depth <= 0 || std::abs(left + right - whole) <= 15.0 * tol) return left + right + (left + right - whole) / 15.0;
        return simpson(a, m, fa, flm, fm, left, 0.5 * tol, depth - 1) +
               simpson(m, b, fm, frm, fb, right, 0.5 * tol, depth - 1);
    }
};

double fill_fraction(const Geometry& g, int w, int i, int j) {
    const double d = g.diameter / g.wfs[static_cast<size_t>(w)].n_subap;
    const double x0 = -g.diameter / 2.0 + j * d;
    const double y0 = -g.diameter / 2.0 + i * d;
    const Cell c{y0, y0 + d, g.r_out(), g.r_in()};
    const double a = x0, b = x0 + d;
    const double fa = c.chord(a), fb = c.chord(b), fm = c.chord(0.5 * (a + b));
    const double whole = (b - a) / 6.0 * (fa + 4.0 * fm + fb);
    return c.simpson(a, b, fa, fm, fb, whole, 1e-12 * d * d, 40) / (d * d);
}

}  // namespace

void validate(const Geometry& g) {
    auto fail = [](const std::string& m) { throw ConfigError("invalid geometry: " + m); };
    if (!(g.diameter > 0.0)) fail("telescope diameter must be > 0");
    if (!(g.obstruction >= 0.0 && g.obstruction < 1.0)) fail("obstruction fraction out of [0,1)");
    if (!(g.threshold > 0.0 && g.threshold <= 1.0)) fail("illumination threshold out of (0,1]");
    if (g.wfs.empty()) fail("wfs list is empty");
    if (g.stars.size() != g.wfs.size())
        fail("guide star count " + std::to_string(g.stars.size()) + " != wfs count " + std::to_string(g.wfs.size()));
    if (g.layers.empty()) fail("layer list is empty");
    if (!g.projection && g.dms.size() != g.layers.size())
        fail("dm count " + std::to_string(g.dms.size()) + " != layer count " + std::to_string(g.layers.size()) +
             " (only the L = M identity-fitting mode is supported)");
    if (g.projection) {
        if (g.dms.empty()) fail("dm list is empty");
        for (const auto& d : g.dms)
            for (int l : d.layers)
                if (l < 0 || l >= static_cast<int>(g.layers.size())) fail("dm layer index out of range");
    }
    for (const auto& w : g.wfs) {
        if (w.n_subap < 1) fail("wfs n_subap must be >= 1");
        if (!(w.noise_variance > 0.0)) fail("wfs noise_variance must be > 0");
    }
    double top = -1.0, sum = 0.0;
    for (const auto& l : g.layers) {
        if (l.height < 0.0) fail("layer height must be >= 0");
        if (l.height <= top) fail("layer heights must be strictly increasing");
        top = l.height;
        if (l.order < 1 || l.order > 16) fail("layer grid_order out of 1..16");
        if (!(l.strength > 0.0 && l.strength <= 1.0)) fail("layer relative_strength out of (0,1]");
        sum += l.strength;
    }
    if (std::abs(sum - 1.0) > 1e-12) fail("layer relative_strength values must sum to 1");
    for (const auto& s : g.stars) {
        if (s.lgs) {
            if (!std::isfinite(s.height) || s.height <= 0.0) fail("LGS height must be finite and > 0");
            if (s.height <= top)
                fail("LGS height " + std::to_string(s.height) + " must exceed top layer height " + std::to_string(top));
        } else if (std::isfinite(s.height)) {
            fail("NGS height must be the infinite marker");
        }
    }
    for (const auto& d : g.dms) {
        if (d.n_act < 2) fail("dm n_act must be >= 2");
        if (d.height < 0.0) fail("dm conjugation height must be >= 0");
    }
    if (!(g.gain >= 0.0 && g.gain <= 1.0)) fail("gain out of [0,1]");
    if (g.pcg_iters < 1) fail("pcg_max_iter must be >= 1");
    if (!(g.pcg_tol >= 0.0 && g.pcg_tol < 1.0)) fail("pcg_tolerance out of [0,1)");
    if (!(g.alpha > 0.0)) fail("regularization alpha must be > 0");
    if (g.wavelet_order < 1 || g.wavelet_order > 10) fail("wavelet order out of 1..10");
    if (!(g.outer_scale > 0.0)) fail("outer scale must be > 0");
    if (!(g.spectral_exponent > 0.0)) fail("spectral exponent must be > 0");
    if (!(g.coarse_weight > 0.0)) fail("preconditioner coarse weight must be > 0");
    if (!(g.balance_exponent >= 0.0 && g.balance_exponent <= 1.0)) fail("preconditioner balance exponent out of [0,1]");
    if (!g.fault.empty() && g.fault != "sh_adjoint") fail("unknown fault fixture '" + g.fault + "'");
    if (g.eval_n_per_side < 1) fail("evaluation grid must be non-empty");
    if (g.eval_half_width < 0.0) fail("evaluation half width must be >= 0");
    if (!(g.truth_strength > 0.0)) fail("simulation truth_strength must be > 0");
    if (!g.wind.empty() && g.wind.size() != g.layers.size()) fail("simulation wind list must have one entry per layer");
    for (size_t l = 0; l < g.layers.size(); ++l) {
        if (g.layers[l].extent > 0.0) {
            const double need_side = meta_pupil(g, static_cast<int>(l));
            if (g.layers[l].extent < need_side * (1.0 - 1e-12))
                fail("layer " + std::to_string(l) + " extent " + std::to_string(g.layers[l].extent) +
                     " below meta-pupil size " + std::to_string(need_side));
        }
    }
}

void finalize(Geometry& g) {
    validate(g);
    for (size_t l = 0; l < g.layers.size(); ++l)
        if (g.layers[l].extent <= 0.0) g.layers[l].extent = derived_extent(g, static_cast<int>(l));
    if (!g.projection) {
        for (size_t m = 0; m < g.dms.size(); ++m) g.dms[m].extent = g.layers[m].extent;  // geometry.hpp:374
    } else {
        bool any_explicit = false;
        for (const auto& d : g.dms) any_explicit = any_explicit || !d.layers.empty();
        if (!any_explicit) {  // default groups: each layer to the DM of nearest conjugation height
            for (size_t l = 0; l < g.layers.size(); ++l) {
                size_t best = 0;
                for (size_t m = 1; m < g.dms.size(); ++m)
                    if (std::abs(g.dms[m].height - g.layers[l].height) < std::abs(g.dms[best].height - g.layers[l].height))
                        best = m;
                g.dms[best].layers.push_back(static_cast<int>(l));
            }
        }
        // DM extent: the reference's layer-extent rule (geometry.hpp:256-275) applied at
        // the DM's conjugation height with its actuator count, so every WFS beam through
        // the DM stays on its grid (add_dm_slopes).  Layers contribute zero to
        // actuators whose projected point falls outside their grid.
        for (auto& d : g.dms) {
            if (d.extent_given) continue;
            double side = 0.0;
            for (const auto& s : g.stars)
                side = std::max(side, s.footprint(d.height) * g.diameter + 2.0 * std::hypot(s.theta_x, s.theta_y) * d.height);
            d.extent = side + 2.0 * side / (d.n_act - 1);
        }
    }
    for (size_t w = 0; w < g.wfs.size(); ++w) {
        const int n = g.wfs[w].n_subap;
        auto& mask = g.wfs[w].mask;
        mask.assign(static_cast<size_t>(n) * n, 0);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                mask[static_cast<size_t>(i) * n + j] =
                    fill_fraction(g, static_cast<int>(w), i, j) >= g.threshold ? 1 : 0;
    }
}

}  // namespace fewha_gpu
