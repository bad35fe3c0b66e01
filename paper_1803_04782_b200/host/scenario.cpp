// scenario.cpp — scenario documents, population seeding and metrics files for the B200 build.
//
// Host-side, one-shot code that keeps the reference's scenario API (proj/src/scenario.cpp) so a
// scenario file and seed produce the same initial SimState: the `key = value` grammar and its
// error behaviour (unknown / duplicate keys rejected with line numbers, scenario.cpp:172-268),
// the constraint checks (:134-170), the canonical serialisation (:278-307), and the placement
// stream — std::mt19937_64 driven through std::uniform_int_distribution<int> and std::shuffle,
// exactly the standard-library types the reference uses (:342-429), so the draws agree under
// the same libstdc++.  The initial strength images are rasterised on the device.

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <map>
#include <random>
#include <sstream>

#include "socfield/scenario.hpp"

namespace socfield {

int direction_count(Directions d) { return static_cast<int>(direction_sects(d).size()); }

std::vector<int> direction_sects(Directions d) {
    switch (d) {
        case Directions::Uni: return {0};
        case Directions::Bi: return {0, 4};
        case Directions::Four: return {0, 2, 4, 6};
        case Directions::Eight: return {0, 1, 2, 3, 4, 5, 6, 7};
    }
    return {};
}

const char* directions_name(Directions d) {
    switch (d) {
        case Directions::Uni: return "uni";
        case Directions::Bi: return "bi";
        case Directions::Four: return "four";
        case Directions::Eight: return "eight";
    }
    return "?";
}

EngineConfig ScenarioConfig::engine_config() const {
    EngineConfig e;
    e.chunk_k = chunk_k;
    e.weight_static = weight_static;
    e.weight_dir_attractive = weight_dir_attractive;
    e.weight_dir_repulsive = weight_dir_repulsive;
    e.weight_recurrent = weight_recurrent;
    e.goal_bias = goal_bias;
    e.regulation = regulation;
    e.density_radius = density_radius;
    e.rebuild_interval = rebuild_interval;
    return e;
}

std::array<FieldSpec, kDynKinds> ScenarioConfig::field_templates() const {
    const auto make = [this](FieldKind kind) { return FieldSpec(kind, field_geometry, field_gain, field_decay, 0); };
    return {make(FieldKind::DirAttractive), make(FieldKind::DirRepulsive), make(FieldKind::RecurrentRepulsive)};
}

// ------------------------------------------------------------------ parsing ----------------

namespace {

std::string strip(const std::string& s) {
    const auto is_space = [](unsigned char c) { return std::isspace(c) != 0; };
    auto first = std::find_if_not(s.begin(), s.end(), is_space);
    auto last = std::find_if_not(s.rbegin(), std::string::const_reverse_iterator(first), is_space).base();
    return std::string(first, last);
}

template <class T, class Conv>
T parse_number(const std::string& text, int line, const char* what, const char* noun, Conv conv) {
    std::size_t used = 0;
    T value{};
    try {
        value = conv(text, &used);
    } catch (const std::exception&) {
        throw ParseError(std::string("expected ") + what + ", got '" + text + "'", line);
    }
    if (used != text.size()) throw ParseError(std::string("trailing characters in ") + noun + " '" + text + "'", line);
    return value;
}

long as_long(const std::string& t, int line) {
    return parse_number<long>(t, line, "an integer", "integer", [](const std::string& s, std::size_t* u) { return std::stol(s, u); });
}
std::uint64_t as_u64(const std::string& t, int line) {
    return parse_number<unsigned long long>(t, line, "an unsigned integer", "integer",
                                            [](const std::string& s, std::size_t* u) { return std::stoull(s, u); });
}
double as_double(const std::string& t, int line) {
    return parse_number<double>(t, line, "a number", "number", [](const std::string& s, std::size_t* u) { return std::stod(s, u); });
}

struct Dims {
    int w, h;
};
Dims as_dims(const std::string& t, int line) {
    const auto x = t.find('x');
    if (x == std::string::npos) throw ParseError("expected WIDTHxHEIGHT, got '" + t + "'", line);
    return Dims{static_cast<int>(as_long(strip(t.substr(0, x)), line)), static_cast<int>(as_long(strip(t.substr(x + 1)), line))};
}

template <class Enum>
Enum as_choice(const std::string& value, const char* field, const char* complaint,
               std::initializer_list<std::pair<const char*, Enum>> options) {
    for (const auto& [name, e] : options)
        if (value == name) return e;
    throw ConfigError(field, complaint);
}

std::string g17(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

using Setter = std::function<void(ScenarioConfig&, const std::string&, int)>;

const std::map<std::string, Setter>& setters() {
    static const std::map<std::string, Setter> table = {
        {"version", [](ScenarioConfig& c, const std::string& v, int l) { c.format_version = static_cast<int>(as_long(v, l)); }},
        {"grid",
         [](ScenarioConfig& c, const std::string& v, int l) {
             const Dims d = as_dims(v, l);
             if (d.w < 1 || d.h < 1) throw ConfigError("grid", "must be at least 1x1");
             c.grid.width = d.w;
             c.grid.height = d.h;
         }},
        {"boundary",
         [](ScenarioConfig& c, const std::string& v, int) {
             c.grid.boundary = as_choice<BoundaryMode>(v, "boundary", "must be 'periodic' or 'closed'",
                                                       {{"periodic", BoundaryMode::Periodic}, {"closed", BoundaryMode::Closed}});
         }},
        {"density", [](ScenarioConfig& c, const std::string& v, int l) { c.density = as_double(v, l); }},
        {"directions",
         [](ScenarioConfig& c, const std::string& v, int) {
             c.directions = as_choice<Directions>(v, "directions", "must be uni, bi, four, or eight",
                                                  {{"uni", Directions::Uni}, {"bi", Directions::Bi},
                                                   {"four", Directions::Four}, {"eight", Directions::Eight}});
         }},
        {"field_geometry",
         [](ScenarioConfig& c, const std::string& v, int l) {
             const Dims d = as_dims(v, l);
             c.field_geometry.width = d.w; // validated as a whole in validate_scenario
             c.field_geometry.height = d.h;
         }},
        {"pedestrian_geometry",
         [](ScenarioConfig& c, const std::string& v, int l) {
             const Dims d = as_dims(v, l);
             c.pedestrian_geometry.width = d.w;
             c.pedestrian_geometry.height = d.h;
         }},
        {"walk_period",
         [](ScenarioConfig& c, const std::string& v, int l) {
             const auto dots = v.find("..");
             if (dots == std::string::npos) {
                 c.walk_period_min = c.walk_period_max = static_cast<int>(as_long(v, l));
             } else {
                 c.walk_period_min = static_cast<int>(as_long(strip(v.substr(0, dots)), l));
                 c.walk_period_max = static_cast<int>(as_long(strip(v.substr(dots + 2)), l));
             }
         }},
        {"chunk_k", [](ScenarioConfig& c, const std::string& v, int l) { c.chunk_k = static_cast<int>(as_long(v, l)); }},
        {"ticks", [](ScenarioConfig& c, const std::string& v, int l) { c.ticks = as_long(v, l); }},
        {"repeats", [](ScenarioConfig& c, const std::string& v, int l) { c.repeats = static_cast<int>(as_long(v, l)); }},
        {"seed", [](ScenarioConfig& c, const std::string& v, int l) { c.seed = as_u64(v, l); }},
        {"field_gain", [](ScenarioConfig& c, const std::string& v, int l) { c.field_gain = as_double(v, l); }},
        {"field_decay", [](ScenarioConfig& c, const std::string& v, int l) { c.field_decay = as_double(v, l); }},
        {"weight_static", [](ScenarioConfig& c, const std::string& v, int l) { c.weight_static = as_double(v, l); }},
        {"weight_dir_attractive", [](ScenarioConfig& c, const std::string& v, int l) { c.weight_dir_attractive = as_double(v, l); }},
        {"weight_dir_repulsive", [](ScenarioConfig& c, const std::string& v, int l) { c.weight_dir_repulsive = as_double(v, l); }},
        {"weight_recurrent", [](ScenarioConfig& c, const std::string& v, int l) { c.weight_recurrent = as_double(v, l); }},
        {"goal_bias", [](ScenarioConfig& c, const std::string& v, int l) { c.goal_bias = as_double(v, l); }},
        {"regulation",
         [](ScenarioConfig& c, const std::string& v, int) {
             c.regulation = as_choice<Regulation>(v, "regulation", "must be 'identity' or 'linear'",
                                                  {{"identity", Regulation::Identity}, {"linear", Regulation::Linear}});
         }},
        {"density_radius", [](ScenarioConfig& c, const std::string& v, int l) { c.density_radius = static_cast<int>(as_long(v, l)); }},
        {"rebuild_interval", [](ScenarioConfig& c, const std::string& v, int l) { c.rebuild_interval = as_long(v, l); }},
    };
    return table;
}

} // namespace

void validate_scenario(const ScenarioConfig& cfg) {
    if (cfg.format_version != 1) throw ConfigError("version", "unsupported format version");
    if (cfg.grid.width < 1 || cfg.grid.height < 1) throw ConfigError("grid", "must be at least 1x1");
    if (!(cfg.density > 0.0) || cfg.density > 1.0) throw ConfigError("density", "must be in (0, 1]");
    const auto odd_positive = [](const Footprint& f) {
        return f.width >= 1 && f.height >= 1 && f.width % 2 == 1 && f.height % 2 == 1;
    };
    if (!odd_positive(cfg.field_geometry)) throw ConfigError("field_geometry", "must be odd x odd");
    if (!odd_positive(cfg.pedestrian_geometry)) throw ConfigError("pedestrian_geometry", "must be odd x odd");
    if (cfg.pedestrian_geometry.width > cfg.grid.width || cfg.pedestrian_geometry.height > cfg.grid.height)
        throw ConfigError("pedestrian_geometry", "must fit inside the grid");
    if (cfg.walk_period_min < 1) throw ConfigError("walk_period", "minimum must be >= 1");
    if (cfg.walk_period_max < cfg.walk_period_min) throw ConfigError("walk_period", "maximum must be >= minimum");
    if (!valid_chunk_width(cfg.chunk_k)) throw ConfigError("chunk_k", "must be 2, 4, 8, or 16");
    if (cfg.ticks < 0) throw ConfigError("ticks", "must be >= 0");
    if (cfg.repeats < 1) throw ConfigError("repeats", "must be >= 1");
    if (!std::isfinite(cfg.field_gain) || !(cfg.field_gain >= 0.0)) throw ConfigError("field_gain", "must be finite and >= 0");
    if (!std::isfinite(cfg.field_decay)) throw ConfigError("field_decay", "must be finite");
    const std::pair<const char*, double> weights[] = {
        {"weight_static", cfg.weight_static},
        {"weight_dir_attractive", cfg.weight_dir_attractive},
        {"weight_dir_repulsive", cfg.weight_dir_repulsive},
        {"weight_recurrent", cfg.weight_recurrent},
        {"goal_bias", cfg.goal_bias},
    };
    for (const auto& [name, value] : weights)
        if (!std::isfinite(value)) throw ConfigError(name, "must be finite");
    if (cfg.density_radius < 0) throw ConfigError("density_radius", "must be >= 0");
    if (cfg.rebuild_interval < 0) throw ConfigError("rebuild_interval", "must be >= 0");
    if (cfg.density * static_cast<double>(cfg.grid.cells()) < static_cast<double>(direction_count(cfg.directions)))
        throw ConfigError("density", "density * grid cells must cover every direction group");
}

ScenarioConfig parse_scenario(const std::string& text) {
    ScenarioConfig cfg;
    std::map<std::string, int> first_seen;
    std::istringstream lines(text);
    std::string raw;
    for (int line = 1; std::getline(lines, raw); ++line) {
        const std::string body = strip(raw.substr(0, raw.find('#')));
        if (body.empty()) continue;
        const auto eq = body.find('=');
        if (eq == std::string::npos) throw ParseError("expected 'key = value'", line);
        const std::string key = strip(body.substr(0, eq));
        const std::string value = strip(body.substr(eq + 1));
        if (key.empty()) throw ParseError("missing key", line);
        if (value.empty()) throw ParseError("missing value for '" + key + "'", line);
        const auto [seen, fresh] = first_seen.try_emplace(key, line);
        if (!fresh)
            throw ParseError("duplicate key '" + key + "' (first on line " + std::to_string(seen->second) + ")", line);
        const auto setter = setters().find(key);
        if (setter == setters().end()) throw ParseError("unknown key '" + key + "'", line);
        setter->second(cfg, value, line);
    }
    validate_scenario(cfg);
    return cfg;
}

ScenarioConfig parse_scenario_file(const std::string& path) {
    std::ifstream file(path);
    if (!file) throw ParseError("cannot open scenario file '" + path + "'");
    std::ostringstream text;
    text << file.rdbuf();
    return parse_scenario(text.str());
}

std::string serialize_scenario(const ScenarioConfig& cfg) {
    std::ostringstream o;
    const auto dims = [](const Footprint& f) { return std::to_string(f.width) + "x" + std::to_string(f.height); };
    o << "version = " << cfg.format_version << '\n'
      << "grid = " << cfg.grid.width << 'x' << cfg.grid.height << '\n'
      << "boundary = " << (cfg.grid.boundary == BoundaryMode::Closed ? "closed" : "periodic") << '\n'
      << "density = " << g17(cfg.density) << '\n'
      << "directions = " << directions_name(cfg.directions) << '\n'
      << "field_geometry = " << dims(cfg.field_geometry) << '\n'
      << "pedestrian_geometry = " << dims(cfg.pedestrian_geometry) << '\n'
      << "walk_period = " << cfg.walk_period_min << ".." << cfg.walk_period_max << '\n'
      << "chunk_k = " << cfg.chunk_k << '\n'
      << "ticks = " << cfg.ticks << '\n'
      << "repeats = " << cfg.repeats << '\n'
      << "seed = " << cfg.seed << '\n'
      << "field_gain = " << g17(cfg.field_gain) << '\n'
      << "field_decay = " << g17(cfg.field_decay) << '\n'
      << "weight_static = " << g17(cfg.weight_static) << '\n'
      << "weight_dir_attractive = " << g17(cfg.weight_dir_attractive) << '\n'
      << "weight_dir_repulsive = " << g17(cfg.weight_dir_repulsive) << '\n'
      << "weight_recurrent = " << g17(cfg.weight_recurrent) << '\n'
      << "goal_bias = " << g17(cfg.goal_bias) << '\n'
      << "regulation = " << (cfg.regulation == Regulation::Linear ? "linear" : "identity") << '\n'
      << "density_radius = " << cfg.density_radius << '\n'
      << "rebuild_interval = " << cfg.rebuild_interval << '\n';
    return o.str();
}

std::int64_t planned_population(const ScenarioConfig& cfg) {
    const double bodies = cfg.density * static_cast<double>(cfg.grid.cells()) / static_cast<double>(cfg.pedestrian_geometry.cells());
    return static_cast<std::int64_t>(std::floor(bodies));
}

Footprint scale_fields(const ScenarioConfig&, int ratio) {
    if (ratio < 1 || ratio % 2 == 0) throw ConfigError("ratio", "must be odd and >= 1");
    return Footprint{7 * ratio, 7 * ratio};
}

// ------------------------------------------------------------------ seeding ----------------

namespace {

// Rejection sampling of non-overlapping centres with a 64-per-pedestrian draw budget, then —
// if the budget runs out — a shuffled footprint-aligned sublattice (scenario.cpp:342-388).
// The order and number of RNG draws is part of the contract: it fixes the initial state.
std::vector<SuIndex> draw_centres(const ScenarioConfig& cfg, std::int64_t want, std::mt19937_64& rng) {
    const GridGeometry& g = cfg.grid;
    const Footprint body = cfg.pedestrian_geometry;
    const int rw = body.half_w(), rh = body.half_h();
    std::vector<SuIndex> centres;
    centres.reserve(static_cast<std::size_t>(want));
    // one bit per su (the reference keeps a 4-byte OccupancyGrid here: 4.3 GB at 32768^2, 134 MB as bits)
    std::vector<std::uint64_t> taken((static_cast<std::size_t>(g.cells()) + 63) / 64, 0);
    const auto bit_of = [&g](SuIndex su) { return static_cast<std::size_t>(su.y) * static_cast<std::size_t>(g.width) + static_cast<std::size_t>(su.x); };
    std::uniform_int_distribution<int> pick_x(0, g.width - 1);
    std::uniform_int_distribution<int> pick_y(0, g.height - 1);

    const auto fits = [&](SuIndex c) {
        if (g.boundary == BoundaryMode::Closed &&
            !(c.x >= rw && c.x + rw < g.width && c.y >= rh && c.y + rh < g.height))
            return false;
        const FootprintCells cells = footprint_cells(g, c, body);
        if (cells.clipped) return false;
        return std::all_of(cells.cells.begin(), cells.cells.end(), [&](SuIndex su) {
            const std::size_t b = bit_of(su);
            return ((taken[b >> 6] >> (b & 63)) & 1u) == 0;
        });
    };

    std::int64_t draws_left = 64 * want;
    bool gave_up = false;
    while (static_cast<std::int64_t>(centres.size()) < want && !gave_up) {
        for (;;) {
            if (draws_left-- <= 0) {
                gave_up = true;
                break;
            }
            const int x = pick_x(rng); // x before y: two separate draws, in this order
            const int y = pick_y(rng);
            const SuIndex c{x, y};
            if (!fits(c)) continue;
            for (const SuIndex su : footprint_cells(g, c, body).cells) {
                const std::size_t b = bit_of(su);
                taken[b >> 6] |= std::uint64_t{1} << (b & 63);
            }
            centres.push_back(c);
            break;
        }
    }
    if (!gave_up) return centres;

    std::vector<SuIndex> lattice;
    for (int y = rh; y + rh < g.height; y += body.height)
        for (int x = rw; x + rw < g.width; x += body.width) lattice.push_back(SuIndex{x, y});
    if (static_cast<std::int64_t>(lattice.size()) < want) {
        throw SeedingError("cannot place " + std::to_string(want) + " pedestrians of " + std::to_string(body.width) +
                           "x" + std::to_string(body.height) + " on a " + std::to_string(g.width) + "x" +
                           std::to_string(g.height) + " grid: density too high for the footprint");
    }
    std::shuffle(lattice.begin(), lattice.end(), rng);
    lattice.resize(static_cast<std::size_t>(want));
    return lattice;
}

} // namespace

std::vector<Pedestrian> seed_pedestrians(const ScenarioConfig& cfg) {
    validate_scenario(cfg);
    const std::int64_t population = planned_population(cfg);

    std::mt19937_64 rng(cfg.seed);
    const std::vector<SuIndex> centres = draw_centres(cfg, population, rng);
    const std::vector<int> goals = direction_sects(cfg.directions);
    const auto templates = cfg.field_templates();
    std::uniform_int_distribution<int> pick_period(cfg.walk_period_min, cfg.walk_period_max);
    const bool fixed_period = cfg.walk_period_min == cfg.walk_period_max;

    std::vector<Pedestrian> pedestrians;
    pedestrians.reserve(centres.size());
    for (std::size_t i = 0; i < centres.size(); ++i) {
        Pedestrian p;
        p.id = static_cast<std::int32_t>(i);
        p.center = centres[i];
        p.footprint = cfg.pedestrian_geometry;
        p.walk_period = fixed_period ? cfg.walk_period_min : pick_period(rng);
        p.walk_phase = static_cast<int>(i) % p.walk_period;
        p.goal_sect = goals[i % goals.size()];
        p.dyn_fields = templates;
        for (FieldSpec& f : p.dyn_fields)
            if (is_directional(f.kind)) f.orientation = p.goal_sect;
        pedestrians.push_back(std::move(p));
    }
    return pedestrians;
}

SimState seed_population(const ScenarioConfig& cfg) {
    SimState state;
    state.pedestrians = seed_pedestrians(cfg);
    state.occupancy = OccupancyGrid(cfg.grid);
    state.static_image = StrengthImage(cfg.grid);
    state.rng_seed = cfg.seed;
    state.tick = 0;
    for (const Pedestrian& p : state.pedestrians)
        for (const SuIndex su : footprint_cells(cfg.grid, p.center, p.footprint).cells) state.occupancy.set(su, p.id);
    state.dyn_images = rasterize_dynamic(state.pedestrians, cfg.grid); // device rasteriser
    return state;
}

// ------------------------------------------------------------------ metrics files -----------

std::size_t write_metrics(const std::vector<TickMetrics>& metrics, std::ostream& out) {
    out << "# socfield-metrics 1\n"
        << "tick,k1_us,k2_us,k3_us,k4_us,k5_us,moved,wall_us\n";
    for (const TickMetrics& m : metrics) {
        out << m.tick;
        for (const std::int64_t us : m.phase_us) out << ',' << us;
        out << ',' << m.moved << ',' << m.wall_us << '\n';
    }
    if (!out) throw std::runtime_error("metrics destination I/O failure");
    return metrics.size();
}

std::size_t write_metrics_file(const std::vector<TickMetrics>& metrics, const std::string& path) {
    std::ofstream file(path);
    if (!file) throw std::runtime_error("cannot open metrics destination '" + path + "'");
    const std::size_t rows = write_metrics(metrics, file);
    file.flush();
    if (!file) throw std::runtime_error("metrics destination I/O failure: '" + path + "'");
    return rows;
}

std::vector<TickMetrics> read_metrics(std::istream& in) {
    std::vector<TickMetrics> rows;
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty() || line.front() == '#' || line.compare(0, 5, "tick,") == 0) continue;
        TickMetrics m;
        long long phase[5];
        const int got = std::sscanf(line.c_str(), "%ld,%lld,%lld,%lld,%lld,%lld,%" SCNd64 ",%" SCNd64, &m.tick, &phase[0],
                                    &phase[1], &phase[2], &phase[3], &phase[4], &m.moved, &m.wall_us);
        if (got != 8) throw ParseError("malformed metrics row: '" + line + "'");
        for (int p = 0; p < 5; ++p) m.phase_us[static_cast<std::size_t>(p)] = phase[p];
        rows.push_back(m);
    }
    return rows;
}

} // namespace socfield
