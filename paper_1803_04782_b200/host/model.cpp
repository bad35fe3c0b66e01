// model.cpp — host side of the socfield model primitives: lattice arithmetic, the strength
// law, write plans, the summation helpers, and the contributor tables handed to the device.
//
// Everything here is construction-time or API-surface code; nothing in this file runs per
// tick.  The numerical pieces (strength_at_offset, sect_index, build_kind_table) deliberately
// evaluate the same expressions with the same libm calls as the reference
// (proj/src/fields.cpp:54-121) because the device consumes their doubles bit for bit.

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "device_bridge.hpp"

namespace socfield {

// ---------------------------------------------------------------- lattice (ref grid.cpp) ----

namespace {
int floor_mod(int value, int modulus) {
    const int r = value % modulus;
    return r >= 0 ? r : r + modulus;
}
} // namespace

GridGeometry::GridGeometry(int w, int h, BoundaryMode b) : width(w), height(h), boundary(b) {
    if (w < 1) throw ConfigError("width", "must be >= 1");
    if (h < 1) throw ConfigError("height", "must be >= 1");
}

Footprint::Footprint(int w, int h) : width(w), height(h) {
    if (w < 1 || (w & 1) == 0) throw ConfigError("footprint.width", "must be odd and positive");
    if (h < 1 || (h & 1) == 0) throw ConfigError("footprint.height", "must be odd and positive");
}

std::optional<SuIndex> wrap(const GridGeometry& g, int x, int y) {
    const bool inside = x >= 0 && x < g.width && y >= 0 && y < g.height;
    if (inside) return SuIndex{x, y};
    if (g.boundary == BoundaryMode::Closed) return std::nullopt;
    return SuIndex{floor_mod(x, g.width), floor_mod(y, g.height)};
}

SuIndex minimal_displacement(const GridGeometry& g, SuIndex center, SuIndex target) {
    SuIndex d{target.x - center.x, target.y - center.y};
    if (g.boundary == BoundaryMode::Closed) return d;
    const auto fold = [](int delta, int extent) {
        const int r = floor_mod(delta, extent);
        return 2 * r > extent ? r - extent : r; // the midpoint keeps its positive image
    };
    d.x = fold(d.x, g.width);
    d.y = fold(d.y, g.height);
    return d;
}

FootprintCells footprint_cells(const GridGeometry& g, SuIndex center, Footprint f) {
    FootprintCells result;
    result.cells.reserve(static_cast<std::size_t>(f.cells()));
    const int rw = f.half_w(), rh = f.half_h();
    for (int dy = -rh; dy <= rh; ++dy) {
        for (int dx = -rw; dx <= rw; ++dx) {
            if (const auto su = wrap(g, center.x + dx, center.y + dy)) result.cells.push_back(*su);
            else result.clipped = true;
        }
    }
    return result;
}

OccupancyGrid::OccupancyGrid(const GridGeometry& g)
    : shape_(g), ids_(static_cast<std::size_t>(g.cells()), kNoPedestrian) {}

std::int64_t OccupancyGrid::occupied_count() const {
    return static_cast<std::int64_t>(
        std::count_if(ids_.begin(), ids_.end(), [](std::int32_t id) { return id != kNoPedestrian; }));
}

double local_density(const OccupancyGrid& occ, SuIndex center, int radius) {
    std::int64_t seen = 0, taken = 0;
    for (int dy = -radius; dy <= radius; ++dy) {
        for (int dx = -radius; dx <= radius; ++dx) {
            const auto su = wrap(occ.geometry(), center.x + dx, center.y + dy);
            if (!su) continue;
            seen += 1;
            taken += occ.empty_at(*su) ? 0 : 1;
        }
    }
    return seen == 0 ? 0.0 : static_cast<double>(taken) / static_cast<double>(seen);
}

// -------------------------------------------------------- summation (ref accumulator.cpp) ----

bool valid_chunk_width(int k) {
    switch (k) {
        case 2: case 4: case 8: case 16: return true;
        default: return false;
    }
}

std::size_t chunk_count(std::size_t n, int k) {
    if (!valid_chunk_width(k)) throw ConfigError("chunk_k", "must be 2, 4, 8, or 16");
    const std::size_t width = static_cast<std::size_t>(k);
    return n / width + (n % width != 0 ? 1 : 0);
}

// ------------------------------------------------------------------ fields (ref fields.cpp) --

bool is_attractive(FieldKind k) { return k == FieldKind::OmniAttractive || k == FieldKind::DirAttractive; }
bool is_directional(FieldKind k) { return k == FieldKind::DirAttractive || k == FieldKind::DirRepulsive; }
bool is_static_kind(FieldKind k) { return k == FieldKind::OmniAttractive || k == FieldKind::OmniRepulsive; }

namespace {
struct KindName {
    FieldKind kind;
    const char* name;
};
constexpr KindName kKindNames[] = {
    {FieldKind::OmniAttractive, "omni-attractive"}, {FieldKind::OmniRepulsive, "omni-repulsive"},
    {FieldKind::DirAttractive, "dir-attractive"},   {FieldKind::DirRepulsive, "dir-repulsive"},
    {FieldKind::RecurrentRepulsive, "recurrent-repulsive"},
};
} // namespace

const char* field_kind_name(FieldKind k) {
    for (const auto& e : kKindNames)
        if (e.kind == k) return e.name;
    return "?";
}

std::optional<FieldKind> field_kind_from_name(const std::string& name) {
    for (const auto& e : kKindNames)
        if (name == e.name) return e.kind;
    return std::nullopt;
}

double Vec2::norm() const { return std::hypot(x, y); }

FieldSpec::FieldSpec(FieldKind kind_, Footprint geometry_, double gain_, double decay_, int orientation_)
    : kind(kind_), geometry(geometry_), gain(gain_), decay(decay_), orientation(orientation_) {
    if (!std::isfinite(gain) || !(gain >= 0.0)) throw ConfigError("gain", "must be finite and >= 0");
    if (!std::isfinite(decay)) throw ConfigError("decay", "must be finite");
    if (orientation < 0 || orientation >= kSects) throw ConfigError("orientation", "must be in [0,8)");
    const double corner = std::hypot(geometry.half_w(), geometry.half_h());
    if (!std::isfinite(gain * std::exp(decay * corner)))
        throw ConfigError("decay", "strength overflows over the field support");
}

int sect_index(Vec2 v) {
    if (v.x == 0.0 && v.y == 0.0) return kNoSect;
    // same expression as the reference: degrees in (-180, 180], wedge s = [45s - 22.5, 45s + 22.5)
    const double deg = std::atan2(v.y, v.x) * 180.0 / M_PI;
    const int wedge = static_cast<int>(std::floor((deg + 22.5) / 45.0));
    return ((wedge % kSects) + kSects) % kSects;
}

int sect_distance(int a, int b) {
    const int forward = (((a - b) % kSects) + kSects) % kSects;
    return std::min(forward, kSects - forward);
}

Offset sect_step(int sect) {
    static constexpr int kDx[kSects] = {1, 1, 0, -1, -1, -1, 0, 1};
    static constexpr int kDy[kSects] = {0, 1, 1, 1, 0, -1, -1, -1};
    return Offset{kDx[sect], kDy[sect]};
}

Vec2 strength_at_offset(const FieldSpec& f, Offset o) {
    const Vec2 none{};
    if (o.dx == 0 && o.dy == 0) return none;
    if (std::abs(o.dx) > f.geometry.half_w() || std::abs(o.dy) > f.geometry.half_h()) return none;
    if (is_directional(f.kind)) {
        const int toward = sect_index(static_cast<double>(o.dx), static_cast<double>(o.dy));
        if (sect_distance(toward, f.orientation) > 1) return none; // outside the 3-sect front cone
    }
    const double r = std::hypot(static_cast<double>(o.dx), static_cast<double>(o.dy));
    const double magnitude = f.gain * std::exp(f.decay * r);
    if (magnitude == 0.0) return none;
    const double sign = is_attractive(f.kind) ? -1.0 : 1.0;
    // evaluation order matters for bit parity with the reference: ((sign*m)*d)/r
    return Vec2{sign * magnitude * o.dx / r, sign * magnitude * o.dy / r};
}

Vec2 strength_at(const FieldSpec& f, SuIndex center, SuIndex target, const GridGeometry& g) {
    const SuIndex d = minimal_displacement(g, center, target);
    return strength_at_offset(f, Offset{d.x, d.y});
}

std::vector<Offset> support(const FieldSpec& f) {
    std::vector<Offset> cells;
    const int rw = f.geometry.half_w(), rh = f.geometry.half_h();
    for (int dy = -rh; dy <= rh; ++dy) {
        for (int dx = -rw; dx <= rw; ++dx) {
            const Vec2 s = strength_at_offset(f, Offset{dx, dy});
            if (s.x != 0.0 || s.y != 0.0) cells.push_back(Offset{dx, dy});
        }
    }
    return cells;
}

namespace detail {

void HostPin::ensure(const void* p, std::size_t bytes) noexcept {
    if (p == ptr_ && bytes == bytes_) return;
    release();
    if (p == nullptr || bytes < (std::size_t{1} << 20)) return;
    if (sfc_host_pin(p, bytes) == 0) {
        ptr_ = p;
        bytes_ = bytes;
    }
}

void HostPin::release() noexcept {
    if (ptr_ != nullptr) sfc_host_unpin(ptr_);
    ptr_ = nullptr;
    bytes_ = 0;
}

} // namespace detail

StrengthImage::StrengthImage(const GridGeometry& g)
    : shape_(g), v_(static_cast<std::size_t>(g.cells()) * kSects, 0.0f) {}

void StrengthImage::clear() { std::fill(v_.begin(), v_.end(), 0.0f); }

float StrengthImage::max_abs_difference(const StrengthImage& a, const StrengthImage& b) {
    float worst = 0.0f;
    const std::size_t n = a.v_.size();
    for (std::size_t i = 0; i != n; ++i) worst = std::max(worst, std::abs(a.v_[i] - b.v_[i]));
    return worst;
}

WritePlan build_write_plan(const FieldSpec& f) {
    WritePlan plan;
    plan.spec_ = f;
    // Walk candidate centre offsets in (dx, dy) order so every per-sect list comes out sorted.
    const int rw = f.geometry.half_w(), rh = f.geometry.half_h();
    for (int cdx = -rw; cdx <= rw; ++cdx) {
        for (int cdy = -rh; cdy <= rh; ++cdy) {
            const Vec2 s = strength_at_offset(f, Offset{-cdx, -cdy}); // target seen from that centre
            if (s.x == 0.0 && s.y == 0.0) continue;
            plan.per_sect_[static_cast<std::size_t>(sect_index(s))].push_back({Offset{cdx, cdy}, s.norm()});
        }
    }
    for (const auto& list : plan.per_sect_) plan.fanout_ = std::max(plan.fanout_, static_cast<int>(list.size()));
    return plan;
}

int fanout_brute_force(const FieldSpec& f) {
    std::array<int, kSects> hits{};
    const int rw = f.geometry.half_w(), rh = f.geometry.half_h();
    for (int cy = -rh; cy <= rh; ++cy) {
        for (int cx = -rw; cx <= rw; ++cx) {
            const Vec2 s = strength_at_offset(f, Offset{-cx, -cy});
            if (s.x != 0.0 || s.y != 0.0) hits[static_cast<std::size_t>(sect_index(s))] += 1;
        }
    }
    return *std::max_element(hits.begin(), hits.end());
}

// ------------------------------------------------------------- device contributor tables ----

namespace bridge {

KindTable build_kind_table(const FieldSpec& spec) {
    KindTable t;
    t.width = spec.geometry.width;
    t.height = spec.geometry.height;
    const int rw = spec.geometry.half_w(), rh = spec.geometry.half_h();
    const std::size_t n = static_cast<std::size_t>(t.width) * static_cast<std::size_t>(t.height);
    t.magnitude.assign(n, 0.0);
    t.info.assign(n, 0u);
    const bool directional = is_directional(spec.kind);
    std::array<std::uint32_t, kSects> rank{}; // next list position per sect
    // (dx, dy) lexicographic over centre offsets == iteration order of the reference's
    // std::map<Offset, GatherEntry>, so `rank` reproduces each entry's list index j.
    for (int cdx = -rw; cdx <= rw; ++cdx) {
        for (int cdy = -rh; cdy <= rh; ++cdy) {
            std::uint32_t mask = 0;
            int sect = 0;
            double magnitude = 0.0;
            for (int orient = 0; orient < (directional ? kSects : 1); ++orient) {
                FieldSpec probe = spec;
                probe.orientation = orient;
                const Vec2 s = strength_at_offset(probe, Offset{-cdx, -cdy});
                if (s.x == 0.0 && s.y == 0.0) continue;
                if (mask == 0) { // the first orientation that reaches the offset fixes the entry
                    sect = sect_index(s);
                    magnitude = s.norm();
                }
                mask |= directional ? (1u << orient) : 0xFFu;
            }
            if (mask == 0) continue;
            const std::size_t at = static_cast<std::size_t>(cdy + rh) * static_cast<std::size_t>(t.width) +
                                   static_cast<std::size_t>(cdx + rw);
            t.magnitude[at] = magnitude;
            t.info[at] = static_cast<std::uint32_t>(sect) | (mask << 3) | (rank[static_cast<std::size_t>(sect)]++ << 11);
        }
    }
    return t;
}

void PedColumns::gather(const std::vector<Pedestrian>& peds) {
    const std::size_t n = peds.size();
    center_xy.resize(2 * n);
    for (auto* col : {&period, &phase, &goal, &orient_a, &orient_r, &foot_w, &foot_h}) col->resize(n);
    for (std::size_t i = 0; i != n; ++i) {
        const Pedestrian& p = peds[i];
        center_xy[2 * i] = p.center.x;
        center_xy[2 * i + 1] = p.center.y;
        period[i] = p.walk_period;
        phase[i] = p.walk_phase;
        goal[i] = p.goal_sect;
        orient_a[i] = p.dyn_fields[0].orientation;
        orient_r[i] = p.dyn_fields[1].orientation;
        foot_w[i] = p.footprint.width;
        foot_h[i] = p.footprint.height;
    }
}

sfc_config make_config(const GridGeometry& g, const EngineConfig& cfg) {
    sfc_config c{};
    c.width = g.width;
    c.height = g.height;
    c.closed = g.boundary == BoundaryMode::Closed ? 1 : 0;
    c.chunk_k = cfg.chunk_k;
    c.weight_static = cfg.weight_static;
    c.weight_dir_attractive = cfg.weight_dir_attractive;
    c.weight_dir_repulsive = cfg.weight_dir_repulsive;
    c.weight_recurrent = cfg.weight_recurrent;
    c.goal_bias = cfg.goal_bias;
    c.regulation = cfg.regulation == Regulation::Linear ? 1 : 0;
    c.density_radius = cfg.density_radius;
    c.rebuild_interval = cfg.rebuild_interval;
    c.rebuild_tolerance = cfg.rebuild_tolerance;
    c.fault_invert_vote_tiebreak = cfg.fault_invert_vote_tiebreak ? 1 : 0;
    c.device = cfg.device;
    // one process per GPU: free functions that build throw-away engines (seeding, rasterize_static)
    // carry no device of their own, so a rank can point them at its GPU with SFC_DEVICE
    if (c.device == 0)
        if (const char* knob = std::getenv("SFC_DEVICE")) c.device = std::atoi(knob);
    c.slab_row0 = 0;
    c.slab_rows = 0;
    return c;
}

void throw_status(int status, const std::string& message, long tick, int phase) {
    switch (status) {
        case SFC_E_INTEGRITY: throw IntegrityError(message, tick, phase);
        case SFC_E_CONFIG: {
            const auto colon = message.find(": ");
            if (colon != std::string::npos) throw ConfigError(message.substr(0, colon), message.substr(colon + 2));
            throw ConfigError("engine", message);
        }
        default: throw std::runtime_error("socfield CUDA engine: " + message);
    }
}

sfc_engine* create_engine(const GridGeometry& g, const EngineConfig& cfg,
                          const std::array<KindTable, kDynKinds>& tables) {
    const sfc_config c = make_config(g, cfg);
    sfc_tables t{};
    for (int k = 0; k < kDynKinds; ++k) t.kind[k] = tables[static_cast<std::size_t>(k)].view();
    sfc_engine* handle = nullptr;
    char why[512] = {0};
    const int status = sfc_create(&c, &t, &handle, why, sizeof why);
    if (status != SFC_OK) throw_status(status, why, -1, 0);
    return handle;
}

} // namespace bridge

} // namespace socfield
