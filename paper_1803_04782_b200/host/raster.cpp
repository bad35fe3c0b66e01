// raster.cpp — the free rasterisation functions of the socfield API, executed on the device:
// rasterize_dynamic (reference engine.cpp:158-168), rasterize_static and rasterize_into
// (fields.cpp:152-168).  The host only prepares contributor tables and item lists.

#include <map>
#include <tuple>

#include "device_bridge.hpp"

namespace socfield {

namespace {

using SpecKey = std::tuple<int, int, int, double, double>; // kind, w, h, gain, decay

SpecKey key_of(const FieldSpec& f) {
    return SpecKey{static_cast<int>(f.kind), f.geometry.width, f.geometry.height, f.gain, f.decay};
}

std::array<bridge::KindTable, kDynKinds> unit_tables() {
    std::array<bridge::KindTable, kDynKinds> t;
    for (int k = 0; k < kDynKinds; ++k)
        t[static_cast<std::size_t>(k)] =
            bridge::build_kind_table(FieldSpec(to_field_kind(static_cast<DynKind>(k)), Footprint{1, 1}));
    return t;
}

struct DeviceHandle {
    sfc_engine* h = nullptr;
    ~DeviceHandle() { sfc_destroy(h); }
};

// Adds `items` (spec, centre) in list order to `base` (or to zeros) in the static image of engine `h`;
// copies the result to `out` when that is not null.
void rasterize_on(sfc_engine* h, const std::vector<AnchoredField>& items, const float* base, float* out) {
    std::map<SpecKey, int> table_of;
    std::vector<bridge::KindTable> storage;
    std::vector<sfc_anchor> anchors;
    anchors.reserve(items.size());
    for (const auto& item : items) {
        auto [it, fresh] = table_of.try_emplace(key_of(item.spec), static_cast<int>(storage.size()));
        if (fresh) storage.push_back(bridge::build_kind_table(item.spec));
        anchors.push_back(sfc_anchor{item.anchor.x, item.anchor.y, it->second,
                                     is_directional(item.spec.kind) ? item.spec.orientation : -1});
    }
    std::vector<sfc_kind_table> views;
    for (const auto& t : storage) views.push_back(t.view());
    const int status = sfc_rasterize_static(h, static_cast<std::int32_t>(views.size()), views.data(),
                                            static_cast<std::int64_t>(anchors.size()), anchors.data(), base, out);
    if (status != SFC_OK) bridge::throw_status(status, sfc_last_error(h), -1, 0);
}

StrengthImage rasterize_list(const GridGeometry& g, const std::vector<AnchoredField>& items, const StrengthImage* base) {
    DeviceHandle dev;
    dev.h = bridge::create_engine(g, EngineConfig{}, unit_tables());
    StrengthImage out(g);
    rasterize_on(dev.h, items, base ? base->raw().data() : nullptr, out.raw_mut().data());
    return out;
}

} // namespace

void bridge::rasterize_static_on(sfc_engine* h, const std::vector<AnchoredField>& fields) {
    rasterize_on(h, fields, nullptr, nullptr);
}

StrengthImage rasterize_static(const std::vector<AnchoredField>& fields, const GridGeometry& g) {
    return rasterize_list(g, fields, nullptr);
}

void rasterize_into(StrengthImage& img, const FieldSpec& f, SuIndex center) {
    img = rasterize_list(img.geometry(), {AnchoredField{f, center}}, &img);
}

std::array<StrengthImage, kDynKinds> rasterize_dynamic(const std::vector<Pedestrian>& pedestrians,
                                                       const GridGeometry& g) {
    std::array<StrengthImage, kDynKinds> images{StrengthImage(g), StrengthImage(g), StrengthImage(g)};
    if (pedestrians.empty()) return images;

    // Fast path: one template per kind slot and one pedestrian per centre — the tiled,
    // id-ordered gather kernel (csrc/sfc_rasterize.cu) handles the whole population at once.
    bool uniform = true;
    OccupancyGrid centres(g);
    for (const Pedestrian& p : pedestrians) {
        for (int k = 0; k < kDynKinds && uniform; ++k) {
            const FieldSpec& mine = p.dyn_fields[static_cast<std::size_t>(k)];
            uniform = mine.kind == to_field_kind(static_cast<DynKind>(k)) &&
                      key_of(mine) == key_of(pedestrians.front().dyn_fields[static_cast<std::size_t>(k)]);
        }
        const auto su = wrap(g, p.center);
        uniform = uniform && su && *su == p.center && centres.empty_at(p.center);
        if (!uniform) break;
        centres.set(p.center, static_cast<std::int32_t>(&p - pedestrians.data()));
    }
    if (uniform) {
        std::array<bridge::KindTable, kDynKinds> tables;
        for (int k = 0; k < kDynKinds; ++k)
            tables[static_cast<std::size_t>(k)] =
                bridge::build_kind_table(pedestrians.front().dyn_fields[static_cast<std::size_t>(k)]);
        DeviceHandle dev;
        dev.h = bridge::create_engine(g, EngineConfig{}, tables);
        // centre-only occupancy with unit footprints: the rasteriser needs centres, not bodies
        std::vector<Pedestrian> points = pedestrians;
        for (std::size_t i = 0; i < points.size(); ++i) {
            points[i].footprint = Footprint{1, 1};
            points[i].walk_period = 1;
            points[i].walk_phase = 0;
        }
        bridge::PedColumns cols;
        cols.gather(points);
        StrengthImage zero(g);
        sfc_state_view v{};
        v.n_peds = static_cast<std::int64_t>(points.size());
        v.occupancy = centres.raw_mut().data();
        v.static_image = zero.raw_mut().data();
        for (int k = 0; k < kDynKinds; ++k) v.dyn_images[k] = images[static_cast<std::size_t>(k)].raw_mut().data();
        v.center_xy = cols.center_xy.data();
        v.walk_period = cols.period.data();
        v.walk_phase = cols.phase.data();
        v.goal_sect = cols.goal.data();
        v.orient_attractive = cols.orient_a.data();
        v.orient_repulsive = cols.orient_r.data();
        v.foot_w = cols.foot_w.data();
        v.foot_h = cols.foot_h.data();
        int status = sfc_upload(dev.h, &v);
        if (status == SFC_OK) {
            float* out[kDynKinds] = {images[0].raw_mut().data(), images[1].raw_mut().data(), images[2].raw_mut().data()};
            status = sfc_rasterize_dynamic(dev.h, out);
        }
        if (status != SFC_OK) bridge::throw_status(status, sfc_last_error(dev.h), -1, 0);
        return images;
    }

    // General path (mixed field specs, shared or unnormalised centres): one ordered device
    // pass per image, items in pedestrian order — the reference's scatter order.
    for (int k = 0; k < kDynKinds; ++k) {
        std::vector<AnchoredField> items;
        items.reserve(pedestrians.size());
        for (const Pedestrian& p : pedestrians) items.push_back(AnchoredField{p.dyn_fields[static_cast<std::size_t>(k)], p.center});
        images[static_cast<std::size_t>(k)] = rasterize_list(g, items, nullptr);
    }
    return images;
}

} // namespace socfield
