// device_bridge.hpp — host-internal helpers shared by the socfield host mirror: building the
// C-ABI contributor tables from FieldSpecs and a small RAII wrapper over sfc_engine.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "socfield/engine.hpp"
#include "socfield_cuda.h"

namespace socfield::bridge {

// Storage behind one sfc_kind_table.
struct KindTable {
    int width = 1, height = 1;
    std::vector<double> magnitude;
    std::vector<std::uint32_t> info;
    sfc_kind_table view() const { return sfc_kind_table{width, height, magnitude.data(), info.data()}; }
};

// Merged contributor table of a field template over all its orientations — the flat form of
// the reference's Engine::build_gather_tables (engine.cpp:201-221); see socfield_cuda.h for
// the bit layout.
KindTable build_kind_table(const FieldSpec& spec);

// SoA copy of the pedestrian attributes an sfc_state_view points into.
struct PedColumns {
    std::vector<std::int32_t> center_xy, period, phase, goal, orient_a, orient_r, foot_w, foot_h;
    void gather(const std::vector<Pedestrian>& peds);
};

sfc_config make_config(const GridGeometry& g, const EngineConfig& cfg);

// Raw-pointer view of a SimState for sfc_upload / sfc_download (cols receives the SoA copy of the
// pedestrian attributes the view points into).
sfc_state_view view_of(SimState& s, PedColumns& cols);

// One row slab of a scenario on one device, stepped from outside (multi-process / multi-GPU runs:
// the caller owns the transport of the halo buffers, see paper_1803_04782_b200/slabs.py).
class SlabEngine {
public:
    SlabEngine(const GridGeometry& g, const EngineConfig& cfg, const std::array<FieldSpec, kDynKinds>& templates,
               int index, int count, int ped_half_h);
    ~SlabEngine();
    SlabEngine(const SlabEngine&) = delete;
    SlabEngine& operator=(const SlabEngine&) = delete;

    void upload(const SimState& s);
    void seed_resident(const std::vector<Pedestrian>& pedestrians, long tick = 0); // no whole-grid host state
    void download(SimState& s);           // writes the rows and pedestrians this slab owns
    void begin(long ticks);
    void step(int which);                 // 0, 1, 2 — see socfield_cuda.h
    std::pair<std::uintptr_t, std::size_t> buffer(int kind, int edge, bool recv);
    std::vector<std::int64_t> finish(long first_tick, long ticks); // synchronises; throws on a device-side error
    int row0() const noexcept { return row0_; }
    int rows() const noexcept { return rows_; }
    int halo() const noexcept { return halo_; }
    bool has_neighbour(int edge) const noexcept;
    sfc_engine* handle() const noexcept { return h_; }

private:
    [[noreturn]] void raise(int status) const;
    sfc_engine* h_ = nullptr;
    GridGeometry geom_;
    int row0_ = 0, rows_ = 0, halo_ = 0;
};

// Throws the socfield exception matching an SFC_E_* status.
[[noreturn]] void throw_status(int status, const std::string& message, long tick, int phase);

// Creates a throw-away engine (whole grid) with the given templates; throws on failure.
sfc_engine* create_engine(const GridGeometry& g, const EngineConfig& cfg,
                          const std::array<KindTable, kDynKinds>& tables);


// rasterize_static(fields) into the static image of a live engine, on its device (no host image).
void rasterize_static_on(sfc_engine* h, const std::vector<AnchoredField>& fields);

} // namespace socfield::bridge
