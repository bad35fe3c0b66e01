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

// Throws the socfield exception matching an SFC_E_* status.
[[noreturn]] void throw_status(int status, const std::string& message, long tick, int phase);

// Creates a throw-away engine (whole grid) with the given templates; throws on failure.
sfc_engine* create_engine(const GridGeometry& g, const EngineConfig& cfg,
                          const std::array<KindTable, kDynKinds>& tables);

} // namespace socfield::bridge
