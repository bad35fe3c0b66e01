// engine.cpp — socfield::Engine of the B200 build: the reference's public engine surface
// (proj/include/socfield/engine.hpp:142-230, proj/src/engine.cpp) as a thin host shim over the
// CUDA C ABI (include/socfield_cuda.h).  No phase of the tick executes on the host.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <thread>

#include "device_bridge.hpp"

namespace socfield {

FieldKind to_field_kind(DynKind k) {
    static constexpr FieldKind kMap[kDynKinds] = {FieldKind::DirAttractive, FieldKind::DirRepulsive,
                                                  FieldKind::RecurrentRepulsive};
    const int i = static_cast<int>(k);
    return i >= 0 && i < kDynKinds ? kMap[i] : FieldKind::RecurrentRepulsive;
}

// Host utility with the reference's semantics (engine.cpp:31-50): descending by score, ties to
// the lower sect.  The device carries its own copy of the 19-comparator network inside k-2;
// this one serves API callers, where any stable ordering with the same key is equivalent.
std::array<int, 8> sort8_desc(const std::array<double, 8>& scores) {
    std::array<int, 8> order{0, 1, 2, 3, 4, 5, 6, 7};
    static constexpr int kNet[19][2] = {{0, 1}, {2, 3}, {0, 2}, {1, 3}, {1, 2}, {4, 5}, {6, 7}, {4, 6}, {5, 7}, {5, 6},
                                        {0, 4}, {1, 5}, {1, 4}, {2, 6}, {3, 7}, {3, 6}, {2, 4}, {3, 5}, {3, 4}};
    for (const auto& wire : kNet) {
        int& hi = order[static_cast<std::size_t>(wire[0])];
        int& lo = order[static_cast<std::size_t>(wire[1])];
        const double sh = scores[static_cast<std::size_t>(hi)], sl = scores[static_cast<std::size_t>(lo)];
        if (sh < sl || (sh == sl && hi > lo)) std::swap(hi, lo);
    }
    return order;
}

// ------------------------------------------------------------------ host mirrors -----------

void EnrollmentTable::reset_geometry(const GridGeometry& g) {
    shape_ = g;
    const std::size_t n = static_cast<std::size_t>(g.cells()) * kSects;
    who_.assign(n, kNoPedestrian);
    how_.assign(n, 0.0);
}

int EnrollmentTable::count(SuIndex su) const {
    const std::size_t first = shape_.flat(su) * kSects;
    return static_cast<int>(std::count_if(who_.begin() + static_cast<std::ptrdiff_t>(first),
                                          who_.begin() + static_cast<std::ptrdiff_t>(first + kSects),
                                          [](std::int32_t id) { return id != kNoPedestrian; }));
}

std::optional<EnrollmentTable::Entry> EnrollmentTable::entry(SuIndex su, int slot) const {
    const std::size_t at = shape_.flat(su) * kSects + static_cast<std::size_t>(slot);
    if (who_[at] == kNoPedestrian) return std::nullopt;
    return Entry{who_[at], how_[at]};
}

void EnrollmentTable::clear_range(std::size_t su_begin, std::size_t su_end) {
    for (std::size_t i = su_begin * kSects; i < su_end * kSects; ++i) {
        who_[i] = kNoPedestrian;
        how_[i] = 0.0;
    }
}

bool EnrollmentTable::enroll(std::size_t su_flat, int slot, std::int32_t id, double score) {
    const std::size_t at = su_flat * kSects + static_cast<std::size_t>(slot);
    if (who_[at] != kNoPedestrian) return false;
    who_[at] = id;
    how_[at] = score;
    return true;
}

void MovementLog::reset(std::size_t cells) {
    moved_from.assign(cells, kNoPedestrian);
    moved_to.assign(cells, kNoPedestrian);
    for (auto& m : from_mask) m.assign(cells, 0);
    for (auto& m : to_mask) m.assign(cells, 0);
}

void MovementLog::clear_range(std::size_t begin, std::size_t end) {
    const auto b = static_cast<std::ptrdiff_t>(begin), e = static_cast<std::ptrdiff_t>(end);
    std::fill(moved_from.begin() + b, moved_from.begin() + e, kNoPedestrian);
    std::fill(moved_to.begin() + b, moved_to.begin() + e, kNoPedestrian);
    for (auto& m : from_mask) std::fill(m.begin() + b, m.begin() + e, std::uint8_t{0});
    for (auto& m : to_mask) std::fill(m.begin() + b, m.begin() + e, std::uint8_t{0});
}

bool states_identical(const SimState& a, const SimState& b, std::string* diagnosis) {
    const auto differ = [diagnosis](const std::string& what) {
        if (diagnosis) *diagnosis = what;
        return false;
    };
    if (a.tick != b.tick) return differ("tick counter differs");
    if (a.pedestrians.size() != b.pedestrians.size()) return differ("pedestrian count differs");
    for (std::size_t i = 0; i < a.pedestrians.size(); ++i) {
        const SuIndex ca = a.pedestrians[i].center, cb = b.pedestrians[i].center;
        if (ca != cb) {
            std::ostringstream msg;
            msg << "pedestrian " << a.pedestrians[i].id << " center (" << ca.x << "," << ca.y << ") vs (" << cb.x
                << "," << cb.y << ")";
            return differ(msg.str());
        }
    }
    const int w = a.occupancy.geometry().width;
    const auto& oa = a.occupancy.raw();
    const auto& ob = b.occupancy.raw();
    if (oa.size() != ob.size()) return differ("occupancy size differs");
    for (std::size_t i = 0; i < oa.size(); ++i) {
        if (oa[i] == ob[i]) continue;
        std::ostringstream msg;
        msg << "occupancy at su (" << i % static_cast<std::size_t>(w) << "," << i / static_cast<std::size_t>(w)
            << "): " << oa[i] << " vs " << ob[i];
        return differ(msg.str());
    }
    // images compare by bit pattern, not by value (-0.0f != 0.0f, NaN == same NaN)
    const auto images_match = [&](const StrengthImage& ia, const StrengthImage& ib, const char* label) {
        const auto& ra = ia.raw();
        const auto& rb = ib.raw();
        if (ra.size() == rb.size() && (ra.empty() || std::memcmp(ra.data(), rb.data(), ra.size() * sizeof(float)) == 0))
            return true;
        const std::size_t n = std::min(ra.size(), rb.size());
        const int iw = ia.geometry().width;
        for (std::size_t i = 0; i < n; ++i) {
            if (std::memcmp(&ra[i], &rb[i], sizeof(float)) == 0) continue;
            const std::size_t su = i / kSects;
            std::ostringstream msg;
            msg << label << " image at su (" << su % static_cast<std::size_t>(iw) << ","
                << su / static_cast<std::size_t>(iw) << ") sect " << i % kSects << ": " << ra[i] << " vs " << rb[i];
            if (diagnosis) *diagnosis = msg.str();
            return false;
        }
        if (diagnosis) *diagnosis = std::string(label) + " image size differs";
        return false;
    };
    if (!images_match(a.static_image, b.static_image, "static")) return false;
    for (int k = 0; k < kDynKinds; ++k) {
        const char* label = field_kind_name(to_field_kind(static_cast<DynKind>(k)));
        if (!images_match(a.dyn_images[static_cast<std::size_t>(k)], b.dyn_images[static_cast<std::size_t>(k)], label))
            return false;
    }
    return true;
}

// ------------------------------------------------------------------ state views ------------

namespace bridge {
sfc_state_view view_of(SimState& s, PedColumns& cols);
}

namespace {

// Pointers into a SimState for the C ABI.  The const_cast on an input-only view is confined to
// the callers: sfc_upload never writes through the pointers.
sfc_state_view make_view(SimState& s, bridge::PedColumns& cols) { return bridge::view_of(s, cols); }

} // namespace

sfc_state_view bridge::view_of(SimState& s, PedColumns& cols) {
    cols.gather(s.pedestrians);
    // the dense arrays cross PCIe on every run: page-lock them once, for as long as their storage lives
    s.occupancy.pin();
    s.static_image.pin();
    for (const StrengthImage& img : s.dyn_images) img.pin();
    sfc_state_view v{};
    v.tick = s.tick;
    v.n_peds = static_cast<std::int64_t>(s.pedestrians.size());
    v.occupancy = s.occupancy.raw_mut().data();
    v.static_image = s.static_image.raw_mut().data();
    for (int k = 0; k < kDynKinds; ++k) v.dyn_images[k] = s.dyn_images[static_cast<std::size_t>(k)].raw_mut().data();
    v.center_xy = cols.center_xy.data();
    v.walk_period = cols.period.data();
    v.walk_phase = cols.phase.data();
    v.goal_sect = cols.goal.data();
    v.orient_attractive = cols.orient_a.data();
    v.orient_repulsive = cols.orient_r.data();
    v.foot_w = cols.foot_w.data();
    v.foot_h = cols.foot_h.data();
    return v;
}

namespace {

void require_shape(const SimState& s, const GridGeometry& g) {
    const std::size_t cells = static_cast<std::size_t>(g.cells());
    if (s.occupancy.raw().size() != cells) throw IntegrityError("occupancy geometry mismatch", s.tick, 0);
    if (s.static_image.raw().size() != cells * kSects) throw IntegrityError("static image geometry mismatch", s.tick, 0);
    for (const auto& img : s.dyn_images)
        if (img.raw().size() != cells * kSects) throw IntegrityError("dynamic image geometry mismatch", s.tick, 0);
}

TickMetrics to_metrics(const sfc_tick_metrics& m) {
    TickMetrics out;
    out.tick = static_cast<long>(m.tick);
    for (int p = 0; p < 5; ++p) out.phase_us[static_cast<std::size_t>(p)] = m.phase_us[p];
    out.moved = m.moved;
    out.wall_us = m.wall_us;
    return out;
}

// The su a step in `direction` newly covers, row-major over the new footprint
// (reference engine.cpp:271-287).  Empty when one falls off a closed grid.
std::vector<SuIndex> newly_covered(const GridGeometry& g, const Pedestrian& p, int direction) {
    std::vector<SuIndex> cells;
    const Offset u = sect_step(direction);
    const int rw = p.footprint.half_w(), rh = p.footprint.half_h();
    for (int oy = -rh; oy <= rh; ++oy) {
        for (int ox = -rw; ox <= rw; ++ox) {
            const bool already = std::abs(ox + u.dx) <= rw && std::abs(oy + u.dy) <= rh;
            if (already) continue;
            const auto su = wrap(g, p.center.x + u.dx + ox, p.center.y + u.dy + oy);
            if (!su) return {};
            cells.push_back(*su);
        }
    }
    return cells;
}

} // namespace

// ------------------------------------------------------------------ Engine -----------------

Engine::Engine(const GridGeometry& g, const EngineConfig& cfg, const std::array<FieldSpec, kDynKinds>& field_templates)
    : geom_(g), cfg_(cfg), field_templates_(field_templates) {
    if (!valid_chunk_width(cfg_.chunk_k)) throw ConfigError("chunk_k", "must be 2, 4, 8, or 16");
    if (cfg_.density_radius < 0) throw ConfigError("density_radius", "must be >= 0");
    if (cfg_.workers <= 0) cfg_.workers = 1; // no host workers exist; keep the field well-formed
    if (const char* knob = std::getenv("SFC_SLABS")) cfg_.slabs = std::atoi(knob); // test hook: force a slab group
    if (cfg_.slabs < 1) throw ConfigError("slabs", "must be >= 1");
    if (const char* knob = std::getenv("SFC_BANDS")) cfg_.bands = std::atoi(knob); // test hook: force a band-swapped run
    if (cfg_.bands < 0) throw ConfigError("bands", "must be >= 0 (0 = as many as the device memory requires)");

    std::array<bridge::KindTable, kDynKinds> tables;
    for (int k = 0; k < kDynKinds; ++k) {
        FieldSpec& spec = field_templates_[static_cast<std::size_t>(k)];
        spec.kind = to_field_kind(static_cast<DynKind>(k));
        auto& plans = plans_[static_cast<std::size_t>(k)];
        if (is_directional(spec.kind)) {
            for (int orient = 0; orient < kSects; ++orient) {
                FieldSpec facing = spec;
                facing.orientation = orient;
                plans.push_back(build_write_plan(facing));
            }
        } else {
            plans.push_back(build_write_plan(spec));
        }
        tables[static_cast<std::size_t>(k)] = bridge::build_kind_table(spec);
    }
    // A banded configuration may describe a state larger than the device's memory: the whole-grid
    // engine is then only built when something other than run() needs it (require_device).
    if (cfg_.bands == 1) dev_ = bridge::create_engine(geom_, cfg_, tables);

    const std::size_t cells = static_cast<std::size_t>(geom_.cells());
    enrollment_.reset_geometry(geom_);
    winners_.assign(cells, kNoPedestrian);
    movelog_.reset(cells);
    step_caches_.assign(1, StepCache(cfg_.chunk_k));
}

Engine::~Engine() {
    release_slabs();
    if (band_engine_) sfc_destroy(band_engine_);
    if (probe_engine_) sfc_destroy(probe_engine_);
    if (dev_) sfc_destroy(dev_);
}

// decide() and rebuild_images() are const probes in the reference; here they upload the state they are
// given.  While the caller steps a resident state (upload / seed_resident ... step_resident) that upload
// must not land on it: the probes then use a scratch engine of their own.
sfc_engine* Engine::probe_device() const {
    require_device();
    if (!resident_live_) return dev_;
    if (!probe_engine_) {
        std::array<bridge::KindTable, kDynKinds> tables;
        for (int k = 0; k < kDynKinds; ++k) tables[static_cast<std::size_t>(k)] = bridge::build_kind_table(field_templates_[static_cast<std::size_t>(k)]);
        probe_engine_ = bridge::create_engine(geom_, cfg_, tables);
    }
    return probe_engine_;
}

void Engine::require_device() const {
    if (dev_) return;
    std::array<bridge::KindTable, kDynKinds> tables;
    for (int k = 0; k < kDynKinds; ++k) tables[static_cast<std::size_t>(k)] = bridge::build_kind_table(field_templates_[static_cast<std::size_t>(k)]);
    const_cast<Engine*>(this)->dev_ = bridge::create_engine(geom_, cfg_, tables);
}

namespace {

// The reference's k-5 adds (float)total to every image address once anybody moved (engine.cpp:468,524), which
// turns a -0.0f entry into +0.0f; the device kernels skip untouched addresses.  Paths that run from host
// state finish with this pass instead (the resident path does it on the device, Ctl::negative_zero).
void normalize_negative_zero(SimState& s, const std::vector<sfc_tick_metrics>& ticks) {
    bool moved = false;
    for (const sfc_tick_metrics& t : ticks) moved = moved || t.moved > 0;
    if (!moved) return;
    for (StrengthImage& img : s.dyn_images)
        for (float& v : img.raw_mut())
            if (v == 0.0f) v = 0.0f; // (-0.0f == 0.0f: rewritten as +0.0f)
}

} // namespace

// run() for a state that does not fit the device: the caller's host SimState is the backing store and
// the SU grid streams through the device in row bands, one phase at a time (sfc_band_run).
std::vector<TickMetrics> Engine::run_bands(SimState& s, long ticks, int bands) {
    int ped_half_h = 0, field_half_h = 0;
    for (const Pedestrian& p : s.pedestrians) ped_half_h = std::max(ped_half_h, p.footprint.half_h());
    for (const FieldSpec& f : field_templates_) field_half_h = std::max(field_half_h, f.geometry.half_h());
    const int halo = sfc_slab_halo_rows(field_half_h, ped_half_h,
                                        cfg_.regulation == Regulation::Linear ? cfg_.density_radius : 0);
    if (bands <= 0) {
        std::int64_t budget = 0; // 0: what the device reports free
        if (const char* knob = std::getenv("SFC_BAND_DEVICE_BYTES")) budget = std::atoll(knob); // plan against a smaller device
        bands = sfc_band_plan(geom_.width, geom_.height, halo, static_cast<std::int64_t>(s.pedestrians.size()), budget, cfg_.device);
        if (bands < 1) throw ConfigError("bands", "the state does not fit the device even in bands one halo tall");
        if (bands == 1) { // it fits: the ordinary resident path
            require_device();
            upload(s);
            std::vector<sfc_tick_metrics> raw(static_cast<std::size_t>(ticks));
            const int status = sfc_run(dev_, ticks, raw.data(), 0);
            download(s);
            resident_live_ = false;
            if (status != SFC_OK) throw_status(status);
            std::vector<TickMetrics> metrics;
            for (const auto& r : raw) metrics.push_back(to_metrics(r));
            return metrics;
        }
    }
    if (bands < 2) throw ConfigError("bands", "a band-swapped run needs at least 2 bands");
    const int rows = (geom_.height + bands - 1) / bands;
    if (!band_engine_ || band_engine_bands_ != bands || slab_halo_ != halo) {
        if (band_engine_) sfc_destroy(band_engine_);
        band_engine_ = nullptr;
        std::array<bridge::KindTable, kDynKinds> tables;
        for (int k = 0; k < kDynKinds; ++k) tables[static_cast<std::size_t>(k)] = bridge::build_kind_table(field_templates_[static_cast<std::size_t>(k)]);
        sfc_tables t{};
        for (int k = 0; k < kDynKinds; ++k) t.kind[k] = tables[static_cast<std::size_t>(k)].view();
        sfc_config c = bridge::make_config(geom_, cfg_);
        c.slab_row0 = 0;
        c.slab_rows = rows;
        c.slab_halo = halo;
        c.bands = (geom_.height + rows - 1) / rows;
        char why[512] = {0};
        const int status = sfc_create(&c, &t, &band_engine_, why, sizeof why);
        if (status != SFC_OK) bridge::throw_status(status, why, s.tick, 0);
        band_engine_bands_ = bands;
        slab_halo_ = halo;
    }
    bridge::PedColumns cols;
    sfc_state_view v = make_view(s, cols);
    std::vector<sfc_tick_metrics> raw(static_cast<std::size_t>(ticks));
    const int status = sfc_band_run(band_engine_, &v, ticks, raw.data());
    normalize_negative_zero(s, raw);
    for (std::size_t i = 0; i < s.pedestrians.size(); ++i) s.pedestrians[i].center = SuIndex{cols.center_xy[2 * i], cols.center_xy[2 * i + 1]};
    s.tick = static_cast<long>(v.tick);
    if (status != SFC_OK) {
        std::int64_t tick = -1;
        std::int32_t phase = 0;
        sfc_error_detail(band_engine_, &tick, &phase, nullptr, nullptr, nullptr);
        bridge::throw_status(status, sfc_last_error(band_engine_), static_cast<long>(tick), phase);
    }
    std::vector<TickMetrics> metrics;
    metrics.reserve(raw.size());
    for (const auto& r : raw) metrics.push_back(to_metrics(r));
    return metrics;
}

void Engine::release_slabs() {
    for (sfc_engine* e : slab_engines_) sfc_destroy(e);
    slab_engines_.clear();
}

// run() over a group of row-slab engines (one per GPU when several are visible): the whole-grid
// host state is scattered over the slabs, the C ABI's group driver steps them with a halo exchange
// per tick, and every slab writes back the rows and pedestrians it owns.
std::vector<TickMetrics> Engine::run_slabs(SimState& s, long ticks) {
    int ped_half_h = 0, field_half_h = 0;
    for (const Pedestrian& p : s.pedestrians) ped_half_h = std::max(ped_half_h, p.footprint.half_h());
    for (const FieldSpec& f : field_templates_) field_half_h = std::max(field_half_h, f.geometry.half_h());
    const int halo = sfc_slab_halo_rows(field_half_h, ped_half_h,
                                        cfg_.regulation == Regulation::Linear ? cfg_.density_radius : 0);
    if (slab_engines_.empty() || halo != slab_halo_) {
        release_slabs();
        const int devices = std::max(1, sfc_device_count());
        std::array<bridge::KindTable, kDynKinds> tables;
        for (int k = 0; k < kDynKinds; ++k) tables[static_cast<std::size_t>(k)] = bridge::build_kind_table(field_templates_[static_cast<std::size_t>(k)]);
        sfc_tables t{};
        for (int k = 0; k < kDynKinds; ++k) t.kind[k] = tables[static_cast<std::size_t>(k)].view();
        for (int i = 0; i < cfg_.slabs; ++i) {
            EngineConfig ec = cfg_;
            ec.device = (cfg_.device + i) % devices;
            sfc_config c = bridge::make_config(geom_, ec);
            c.slab_row0 = static_cast<std::int32_t>(static_cast<std::int64_t>(geom_.height) * i / cfg_.slabs);
            c.slab_rows = static_cast<std::int32_t>(static_cast<std::int64_t>(geom_.height) * (i + 1) / cfg_.slabs) - c.slab_row0;
            c.slab_halo = halo;
            sfc_engine* handle = nullptr;
            char why[512] = {0};
            const int status = sfc_create(&c, &t, &handle, why, sizeof why);
            if (status != SFC_OK) {
                release_slabs();
                bridge::throw_status(status, why, s.tick, 0);
            }
            slab_engines_.push_back(handle);
        }
        slab_halo_ = halo;
    }
    bridge::PedColumns cols;
    sfc_state_view v = make_view(s, cols);
    const auto fail_with = [&](sfc_engine* e, int status) {
        std::int64_t tick = -1;
        std::int32_t phase = 0;
        sfc_error_detail(e, &tick, &phase, nullptr, nullptr, nullptr);
        bridge::throw_status(status, sfc_last_error(e), static_cast<long>(tick), phase);
    };
    for (sfc_engine* e : slab_engines_) {
        const int status = sfc_upload(e, &v);
        if (status != SFC_OK) fail_with(e, status);
    }
    std::vector<sfc_tick_metrics> raw(static_cast<std::size_t>(ticks));
    const int run_status = sfc_group_run(slab_engines_.data(), static_cast<int>(slab_engines_.size()), ticks, raw.data());
    v.static_image = nullptr;
    for (sfc_engine* e : slab_engines_) {
        const int status = sfc_download(e, &v);
        if (status != SFC_OK) fail_with(e, status);
    }
    if (run_status == SFC_OK) normalize_negative_zero(s, raw);
    for (std::size_t i = 0; i < s.pedestrians.size(); ++i) s.pedestrians[i].center = SuIndex{cols.center_xy[2 * i], cols.center_xy[2 * i + 1]};
    s.tick = static_cast<long>(v.tick);
    if (run_status != SFC_OK) fail_with(slab_engines_.front(), run_status);
    std::vector<TickMetrics> metrics;
    metrics.reserve(raw.size());
    for (const auto& r : raw) metrics.push_back(to_metrics(r));
    return metrics;
}

const WritePlan& Engine::plan(DynKind kind, int orientation) const {
    const auto& plans = plans_[static_cast<std::size_t>(kind)];
    if (plans.size() == 1) return plans.front();
    return plans.at(static_cast<std::size_t>(orientation));
}

void Engine::throw_status(int status) const {
    std::int64_t tick = -1;
    std::int32_t phase = 0;
    sfc_error_detail(dev_, &tick, &phase, nullptr, nullptr, nullptr);
    bridge::throw_status(status, sfc_last_error(dev_), static_cast<long>(tick), phase);
}

void Engine::upload(const SimState& s) {
    require_device();
    require_shape(s, geom_);
    bridge::PedColumns cols;
    const sfc_state_view v = make_view(const_cast<SimState&>(s), cols);
    const int status = sfc_upload(dev_, &v);
    if (status != SFC_OK) throw_status(status);
    resident_live_ = true; // (run() / tick() clear it again: after their download the host state is authoritative)
    if (decisions_.size() != s.pedestrians.size()) decisions_.assign(s.pedestrians.size(), kStill);
}

void Engine::download(SimState& s) {
    require_device();
    bridge::PedColumns cols;
    sfc_state_view v = make_view(s, cols);
    v.static_image = nullptr; // a tick never writes it
    const int status = sfc_download(dev_, &v);
    if (status != SFC_OK) throw_status(status);
    for (std::size_t i = 0; i < s.pedestrians.size(); ++i)
        s.pedestrians[i].center = SuIndex{cols.center_xy[2 * i], cols.center_xy[2 * i + 1]};
    s.tick = static_cast<long>(v.tick);
}

namespace {
// A state view that carries the pedestrians only: sfc_upload then builds the dense buffers on the device.
sfc_state_view population_view(const std::vector<Pedestrian>& peds, long tick, bridge::PedColumns& cols) {
    cols.gather(peds);
    sfc_state_view v{};
    v.tick = tick;
    v.n_peds = static_cast<std::int64_t>(peds.size());
    v.center_xy = cols.center_xy.data();
    v.walk_period = cols.period.data();
    v.walk_phase = cols.phase.data();
    v.goal_sect = cols.goal.data();
    v.orient_attractive = cols.orient_a.data();
    v.orient_repulsive = cols.orient_r.data();
    v.foot_w = cols.foot_w.data();
    v.foot_h = cols.foot_h.data();
    return v;
}
} // namespace

void Engine::seed_resident(const std::vector<Pedestrian>& pedestrians, long tick) {
    require_device();
    bridge::PedColumns cols;
    const sfc_state_view v = population_view(pedestrians, tick, cols);
    const int status = sfc_upload(dev_, &v);
    if (status != SFC_OK) throw_status(status);
    resident_live_ = true;
    decisions_.assign(pedestrians.size(), kStill);
}

std::vector<SuIndex> Engine::download_centers() {
    require_device();
    std::vector<std::int32_t> xy(2 * decisions_.size());
    sfc_state_view v{};
    v.n_peds = static_cast<std::int64_t>(decisions_.size());
    v.center_xy = xy.data();
    const int status = sfc_download(dev_, &v);
    if (status != SFC_OK) throw_status(status);
    std::vector<SuIndex> out(decisions_.size());
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = SuIndex{xy[2 * i], xy[2 * i + 1]};
    return out;
}

void Engine::set_static_resident(const std::vector<AnchoredField>& fields) {
    require_device();
    bridge::rasterize_static_on(dev_, fields);
}

std::uint64_t Engine::digest_resident() {
    require_device();
    std::uint64_t h = 0;
    const int status = sfc_digest(dev_, &h);
    if (status != SFC_OK) throw_status(status);
    return h;
}

bool Engine::resident_identical(Engine& other, std::string* diagnosis) { // wording of states_identical, engine.cpp:103-156
    sfc_difference d{};
    require_device();
    other.require_device();
    const int status = sfc_compare(dev_, other.dev_, &d);
    if (status != SFC_OK) throw_status(status);
    if (d.what == 0) return true;
    std::ostringstream os;
    const long w = geom_.width;
    if (d.what == 1) os << "tick counter differs";
    else if (d.what == 2) os << "pedestrian count differs";
    else if (d.what == 3)
        os << "pedestrian " << d.index << " center (" << d.ax << "," << d.ay << ") vs (" << d.bx << "," << d.by << ")";
    else if (d.what == 4) os << "occupancy at su (" << d.index % w << "," << d.index / w << "): " << d.ax << " vs " << d.bx;
    else {
        const char* name = d.what == 5 ? "static" : field_kind_name(to_field_kind(static_cast<DynKind>(d.what - 6)));
        os << name << " image at su (" << (d.index / kSects) % w << "," << (d.index / kSects) / w << ") sect " << d.index % kSects
           << ": " << d.av << " vs " << d.bv;
    }
    if (diagnosis) *diagnosis = os.str();
    return false;
}

std::vector<TickMetrics> Engine::step_resident(long ticks, bool phase_times) {
    require_device();
    std::vector<TickMetrics> out;
    if (ticks <= 0) return out;
    std::vector<sfc_tick_metrics> raw(static_cast<std::size_t>(ticks));
    const int status = sfc_run(dev_, ticks, raw.data(), phase_times ? 1 : 0);
    if (status != SFC_OK) throw_status(status);
    out.reserve(raw.size());
    for (const auto& m : raw) out.push_back(to_metrics(m));
    return out;
}

void Engine::pull_temporaries(int phase, SimState& s) {
    require_device();
    const std::size_t cells = static_cast<std::size_t>(geom_.cells());
    std::vector<std::uint8_t> from(3 * cells), to(3 * cells);
    std::vector<std::int32_t> dirs(s.pedestrians.size());
    sfc_temporaries t{};
    t.decisions = dirs.data();
    t.enroll_ids = enrollment_.ids_mut().data();
    t.enroll_scores = enrollment_.scores_mut().data();
    t.winners = winners_.data();
    t.moved_from = movelog_.moved_from.data();
    t.moved_to = movelog_.moved_to.data();
    t.from_mask = from.data();
    t.to_mask = to.data();
    const int status = sfc_download_temporaries(dev_, &t);
    if (status != SFC_OK) throw_status(status);
    for (int k = 0; k < kDynKinds; ++k) {
        const auto b = static_cast<std::ptrdiff_t>(static_cast<std::size_t>(k) * cells);
        const auto e = b + static_cast<std::ptrdiff_t>(cells);
        movelog_.from_mask[static_cast<std::size_t>(k)].assign(from.begin() + b, from.begin() + e);
        movelog_.to_mask[static_cast<std::size_t>(k)].assign(to.begin() + b, to.begin() + e);
    }
    decisions_.assign(dirs.begin(), dirs.end());
    if (phase >= 4) {
        const long tick_before = s.tick;
        download(s);
        resident_live_ = false;
        s.tick = tick_before; // the counter advances only at the end of the tick
    }
}

TickMetrics Engine::tick(SimState& s, RunMode mode) { return tick(s, mode, Inspector{}); }

TickMetrics Engine::tick(SimState& s, RunMode /*mode*/, const Inspector& inspect) {
    require_device();
    upload(s);
    TickMetrics m;
    m.tick = s.tick;
    if (!inspect) {
        int status = SFC_OK;
        sfc_tick_metrics raw{};
        status = sfc_run(dev_, 1, &raw, 1);
        download(s); // the state is meaningful even when the tick ended in an integrity error
        resident_live_ = false;
        if (status != SFC_OK) throw_status(status);
        return to_metrics(raw);
    }
    // Inspector path: one phase at a time, host mirrors refreshed after each (engine.cpp:487-530).
    for (int phase = 1; phase <= 5; ++phase) {
        std::int64_t moved = 0;
        const int status = sfc_phase(dev_, phase, phase >= 4 ? &moved : nullptr);
        if (status != SFC_OK) {
            download(s);
            resident_live_ = false;
            throw_status(status);
        }
        if (phase >= 4) m.moved = moved;
        pull_temporaries(phase, s);
        inspect(phase, *this, s);
    }
    const int status = sfc_phase(dev_, 6, nullptr);
    download(s);
    resident_live_ = false;
    if (status != SFC_OK) throw_status(status);
    return m;
}

std::vector<TickMetrics> Engine::run(SimState& s, long ticks, RunMode mode) { return run(s, ticks, mode, Inspector{}); }

std::vector<TickMetrics> Engine::run(SimState& s, long ticks, RunMode mode, const Inspector& inspect) {
    std::vector<TickMetrics> metrics;
    if (ticks <= 0 || inspect || cfg_.slabs > 1 || cfg_.bands != 1) {
        verify_state(s);
        if (ticks <= 0) return metrics;
        if (inspect) {
            metrics.reserve(static_cast<std::size_t>(ticks));
            for (long i = 0; i < ticks; ++i) metrics.push_back(tick(s, mode, inspect));
            return metrics;
        }
        if (cfg_.slabs > 1) return run_slabs(s, ticks);
        return run_bands(s, ticks, cfg_.bands);
    }
    {   // verify_state (host, ~1 ms per million su) runs while the state is on its way to the device; a
        // rejected state throws before any tick runs, exactly as if it had been checked first
        std::exception_ptr rejected, upload_failed;
        std::thread checker([&] {
            try {
                verify_state(s);
            } catch (...) {
                rejected = std::current_exception();
            }
        });
        try {
            upload(s);
        } catch (...) {
            upload_failed = std::current_exception();
        }
        checker.join();
        if (rejected) std::rethrow_exception(rejected);
        if (upload_failed) std::rethrow_exception(upload_failed);
    }
    std::vector<sfc_tick_metrics> raw(static_cast<std::size_t>(ticks));
    const int status = sfc_run(dev_, ticks, raw.data(), 0);
    download(s);
    resident_live_ = false;
    if (status != SFC_OK) throw_status(status);
    metrics.reserve(raw.size());
    for (const auto& r : raw) metrics.push_back(to_metrics(r));
    return metrics;
}

MoveDecision Engine::decide(const Pedestrian& p, const SimState& s) const {
    require_device();
    require_shape(s, geom_);
    // The device decides for the pedestrian stored at p.id; substitute `p` there so callers may
    // probe a modified copy, as the reference's by-value semantics allow.
    SimState probe = s;
    const std::size_t slot = static_cast<std::size_t>(p.id);
    if (slot >= probe.pedestrians.size()) throw IntegrityError("decide: pedestrian id out of range", s.tick, 0);
    probe.pedestrians[slot] = p;
    bridge::PedColumns cols;
    const sfc_state_view v = make_view(probe, cols);
    sfc_engine* const dev = probe_device();
    int status = sfc_upload(dev, &v);
    if (status != SFC_OK) bridge::throw_status(status, sfc_last_error(dev), s.tick, 0);
    MoveDecision d;
    std::int32_t dir = kStill;
    status = sfc_decide(dev, p.id, &dir, &d.score);
    if (status != SFC_OK) bridge::throw_status(status, sfc_last_error(dev), s.tick, 2);
    d.direction = dir;
    if (dir != kStill) d.new_cells = newly_covered(geom_, p, dir);
    return d;
}

std::array<StrengthImage, kDynKinds> Engine::rebuild_images(const SimState& s) const {
    require_device();
    require_shape(s, geom_);
    bridge::PedColumns cols;
    const sfc_state_view v = make_view(const_cast<SimState&>(s), cols);
    sfc_engine* const dev = probe_device();
    int status = sfc_upload(dev, &v);
    if (status != SFC_OK) bridge::throw_status(status, sfc_last_error(dev), s.tick, 0);
    std::array<StrengthImage, kDynKinds> fresh{StrengthImage(geom_), StrengthImage(geom_), StrengthImage(geom_)};
    float* out[kDynKinds] = {fresh[0].raw_mut().data(), fresh[1].raw_mut().data(), fresh[2].raw_mut().data()};
    status = sfc_rasterize_dynamic(dev, out);
    if (status != SFC_OK) bridge::throw_status(status, sfc_last_error(dev), s.tick, 0);
    return fresh;
}

// Structural check of a host state (reference engine.cpp:569-618).  Integer bookkeeping on the
// caller's own buffers; it guards the upload, it is not part of the tick.
void Engine::verify_state(const SimState& s) const {
    const auto reject = [&s](const std::string& what) { throw IntegrityError(what, s.tick, 0); };
    if (!(s.occupancy.geometry() == geom_)) reject("occupancy geometry mismatch");
    {   // Fast acceptance of a consistent state (every run() starts here): each pedestrian is well-formed and
        // every su of its body holds its id, and the grid holds no other occupant.  Anything else falls
        // through to the reference's check below, which finds the FIRST violation in its order and words it.
        const auto& occ = s.occupancy.raw();
        const std::size_t w = static_cast<std::size_t>(geom_.width);
        bool fine = true;
        std::size_t body_cells = 0;
        for (std::size_t i = 0; i < s.pedestrians.size() && fine; ++i) {
            const Pedestrian& p = s.pedestrians[i];
            fine = p.id == static_cast<std::int32_t>(i) && p.center.x >= 0 && p.center.x < geom_.width && p.center.y >= 0 &&
                   p.center.y < geom_.height && p.walk_period >= 1 && p.walk_phase >= 0 && p.walk_phase < p.walk_period &&
                   p.goal_sect >= 0 && p.goal_sect < kSects;
            for (int k = 0; k < kDynKinds && fine; ++k) {
                const FieldSpec& have = p.dyn_fields[static_cast<std::size_t>(k)];
                const FieldSpec& want = field_templates_[static_cast<std::size_t>(k)];
                fine = have.kind == want.kind && have.geometry == want.geometry && have.gain == want.gain && have.decay == want.decay;
            }
            if (!fine) break;
            if (p.footprint.width == 1 && p.footprint.height == 1) {
                fine = occ[static_cast<std::size_t>(p.center.y) * w + static_cast<std::size_t>(p.center.x)] == p.id;
                body_cells += 1;
            } else {
                const FootprintCells body = footprint_cells(geom_, p.center, p.footprint);
                fine = !body.clipped;
                for (const SuIndex su : body.cells) fine = fine && s.occupancy.at(su) == p.id;
                body_cells += body.cells.size();
            }
        }
        if (fine) {
            std::size_t occupied = 0;
            for (const std::int32_t id : occ) occupied += id != kNoPedestrian;
            if (occupied == body_cells) return; // (a body wrapping onto itself repeats su: counts differ, slow path words it)
        }
    }
    OccupancyGrid expected(geom_);
    for (std::size_t i = 0; i < s.pedestrians.size(); ++i) {
        const Pedestrian& p = s.pedestrians[i];
        const auto who = [&p] { return "pedestrian " + std::to_string(p.id); }; // (only built for a rejection)
        if (p.id != static_cast<std::int32_t>(i)) reject("pedestrian ids must equal their index");
        const auto normal = wrap(geom_, p.center);
        if (!normal || *normal != p.center) reject(who() + " center not normalized");
        if (p.walk_period < 1 || p.walk_phase < 0 || p.walk_phase >= p.walk_period) reject(who() + " walk gate out of range");
        if (p.goal_sect < 0 || p.goal_sect >= kSects) reject(who() + " goal sect out of range");
        for (int k = 0; k < kDynKinds; ++k) {
            const FieldSpec& have = p.dyn_fields[static_cast<std::size_t>(k)];
            const FieldSpec& want = field_templates_[static_cast<std::size_t>(k)];
            if (have.kind != want.kind || have.geometry != want.geometry || have.gain != want.gain ||
                have.decay != want.decay)
                reject(who() + " field spec does not match the engine template");
        }
        const FootprintCells body = footprint_cells(geom_, p.center, p.footprint);
        if (body.clipped) reject(who() + " footprint crosses a closed edge");
        for (const SuIndex su : body.cells) {
            if (!expected.empty_at(su)) {
                if (expected.at(su) == p.id) reject(who() + " footprint wraps onto itself");
                reject("pedestrians " + std::to_string(expected.at(su)) + " and " + std::to_string(p.id) +
                       " overlap at su (" + std::to_string(su.x) + "," + std::to_string(su.y) + ")");
            }
            expected.set(su, p.id);
        }
    }
    const auto& got = s.occupancy.raw();
    const auto& want = expected.raw();
    if (got.size() == want.size() && std::memcmp(got.data(), want.data(), got.size() * sizeof(got[0])) == 0) return;
    for (std::size_t i = 0; i < got.size(); ++i) {
        if (got[i] == want[i]) continue;
        const std::size_t w = static_cast<std::size_t>(geom_.width);
        reject("occupancy at su (" + std::to_string(i % w) + "," + std::to_string(i / w) + ") holds " +
               std::to_string(got[i]) + ", expected " + std::to_string(want[i]));
    }
}

} // namespace socfield

// ------------------------------------------------------------------ SlabEngine --------------

namespace socfield::bridge {

SlabEngine::SlabEngine(const GridGeometry& g, const EngineConfig& cfg, const std::array<FieldSpec, kDynKinds>& templates,
                       int index, int count, int ped_half_h)
    : geom_(g) {
    if (count < 2 || index < 0 || index >= count) throw ConfigError("slabs", "need 0 <= index < count and count >= 2");
    std::array<KindTable, kDynKinds> tables;
    int field_half_h = 0;
    for (int k = 0; k < kDynKinds; ++k) {
        FieldSpec spec = templates[static_cast<std::size_t>(k)];
        spec.kind = to_field_kind(static_cast<DynKind>(k));
        tables[static_cast<std::size_t>(k)] = build_kind_table(spec);
        field_half_h = std::max(field_half_h, spec.geometry.half_h());
    }
    halo_ = sfc_slab_halo_rows(field_half_h, ped_half_h, cfg.regulation == Regulation::Linear ? cfg.density_radius : 0);
    row0_ = static_cast<int>(static_cast<std::int64_t>(g.height) * index / count);
    rows_ = static_cast<int>(static_cast<std::int64_t>(g.height) * (index + 1) / count) - row0_;
    sfc_config c = make_config(g, cfg);
    c.slab_row0 = row0_;
    c.slab_rows = rows_;
    c.slab_halo = halo_;
    sfc_tables t{};
    for (int k = 0; k < kDynKinds; ++k) t.kind[k] = tables[static_cast<std::size_t>(k)].view();
    char why[512] = {0};
    const int status = sfc_create(&c, &t, &h_, why, sizeof why);
    if (status != SFC_OK) throw_status(status, why, -1, 0);
}

SlabEngine::~SlabEngine() { sfc_destroy(h_); }

void SlabEngine::raise(int status) const {
    std::int64_t tick = -1;
    std::int32_t phase = 0;
    sfc_error_detail(h_, &tick, &phase, nullptr, nullptr, nullptr);
    throw_status(status, sfc_last_error(h_), static_cast<long>(tick), phase);
}

bool SlabEngine::has_neighbour(int edge) const noexcept {
    if (geom_.boundary == BoundaryMode::Periodic) return true;
    return edge == 0 ? row0_ > 0 : row0_ + rows_ < geom_.height;
}

void SlabEngine::upload(const SimState& s) {
    PedColumns cols;
    const sfc_state_view v = view_of(const_cast<SimState&>(s), cols);
    const int status = sfc_upload(h_, &v);
    if (status != SFC_OK) raise(status);
}

void SlabEngine::seed_resident(const std::vector<Pedestrian>& pedestrians, long tick) {
    PedColumns cols;
    cols.gather(pedestrians);
    sfc_state_view v{};
    v.tick = tick;
    v.n_peds = static_cast<std::int64_t>(pedestrians.size());
    v.center_xy = cols.center_xy.data();
    v.walk_period = cols.period.data();
    v.walk_phase = cols.phase.data();
    v.goal_sect = cols.goal.data();
    v.orient_attractive = cols.orient_a.data();
    v.orient_repulsive = cols.orient_r.data();
    v.foot_w = cols.foot_w.data();
    v.foot_h = cols.foot_h.data();
    const int status = sfc_upload(h_, &v);
    if (status != SFC_OK) raise(status);
}

void SlabEngine::download(SimState& s) {
    PedColumns cols;
    sfc_state_view v = view_of(s, cols);
    v.static_image = nullptr;
    const int status = sfc_download(h_, &v);
    if (status != SFC_OK) raise(status);
    for (std::size_t i = 0; i < s.pedestrians.size(); ++i)
        s.pedestrians[i].center = SuIndex{cols.center_xy[2 * i], cols.center_xy[2 * i + 1]};
    s.tick = static_cast<long>(v.tick);
}

void SlabEngine::begin(long ticks) {
    const int status = sfc_slab_begin(h_, ticks);
    if (status != SFC_OK) raise(status);
}

void SlabEngine::step(int which) {
    const int status = sfc_slab_step(h_, which);
    if (status != SFC_OK) raise(status);
}

std::pair<std::uintptr_t, std::size_t> SlabEngine::buffer(int kind, int edge, bool recv) {
    void* ptr = nullptr;
    std::size_t bytes = 0;
    const int status = sfc_slab_buffer(h_, kind, edge, recv ? 1 : 0, &ptr, &bytes);
    if (status != SFC_OK) raise(status);
    return {reinterpret_cast<std::uintptr_t>(ptr), bytes};
}

std::vector<std::int64_t> SlabEngine::finish(long first_tick, long ticks) {
    std::vector<std::int64_t> moved(static_cast<std::size_t>(std::max(0L, ticks)));
    const int status = sfc_slab_finish(h_, first_tick, ticks, moved.data());
    if (status != SFC_OK) raise(status);
    return moved;
}

} // namespace socfield::bridge
