// socfield_shim.cpp — see socfield_shim.h.  TEST INFRASTRUCTURE.
//
// Written only against the public socfield C++ API (socfield/scenario.hpp pulls in
// engine.hpp, fields.hpp, grid.hpp, accumulator.hpp, errors.hpp), so that it compiles
// unchanged against the reference tree and against this repository's host mirror.
// Compile with -DSHIM_IMPL_NAME=\"...\" to label the build.

#include "socfield_shim.h"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "socfield/scenario.hpp"

#ifndef SHIM_IMPL_NAME
#define SHIM_IMPL_NAME "unknown"
#endif

using namespace socfield;

struct shim_sim {
    GridGeometry grid;
    EngineConfig ecfg;
    std::array<FieldSpec, kDynKinds> templates;
    std::unique_ptr<Engine> engine;
    SimState state;
};

namespace {

void put_err(char* err, size_t errlen, const std::string& msg) {
    if (!err || errlen == 0) return;
    std::snprintf(err, errlen, "%s", msg.c_str());
}

// Maps the API's exception taxonomy (errors.hpp) onto the shim's return codes.
template <class Fn>
int guarded(char* err, size_t errlen, Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const IntegrityError& e) {
        put_err(err, errlen, e.what());
        return 1;
    } catch (const ConfigError& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const ParseError& e) {
        put_err(err, errlen, e.what());
        return 3;
    } catch (const SeedingError& e) {
        put_err(err, errlen, e.what());
        return 4;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 5;
    }
}

std::size_t cell_count(const shim_sim* s) { return static_cast<std::size_t>(s->grid.cells()); }

RunMode run_mode(int mode) { return mode == 0 ? RunMode::Sequential : RunMode::Parallel; }

StrengthImage& image_ref(shim_sim* s, int which) {
    return which < 0 ? s->state.static_image : s->state.dyn_images[static_cast<std::size_t>(which)];
}

std::uint64_t fnv1a(const void* data, std::size_t bytes, std::uint64_t h) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

void capture_phase(int phase, const Engine& e, const SimState& st, shim_capture* cap) {
    const std::size_t cells = static_cast<std::size_t>(st.occupancy.geometry().cells());
    const std::size_t peds = st.pedestrians.size();
    cap->phases_seen |= (1 << phase);
    if (phase == 2) {
        if (cap->decisions)
            for (std::size_t i = 0; i < peds; ++i) cap->decisions[i] = e.decision_direction(i);
        if (cap->enroll_ids || cap->enroll_scores) {
            for (std::size_t su = 0; su < cells; ++su) {
                for (int slot = 0; slot < kSects; ++slot) {
                    if (cap->enroll_ids) cap->enroll_ids[su * kSects + slot] = e.enrollment().id_at(su, slot);
                    if (cap->enroll_scores)
                        cap->enroll_scores[su * kSects + slot] = e.enrollment().score_at(su, slot);
                }
            }
        }
    } else if (phase == 3) {
        if (cap->winners) std::copy(e.vote_winners().begin(), e.vote_winners().end(), cap->winners);
    } else if (phase == 4) {
        const MovementLog& log = e.movement_log();
        if (cap->moved_from) std::copy(log.moved_from.begin(), log.moved_from.end(), cap->moved_from);
        if (cap->moved_to) std::copy(log.moved_to.begin(), log.moved_to.end(), cap->moved_to);
        for (int k = 0; k < kDynKinds; ++k) {
            if (cap->from_mask)
                std::copy(log.from_mask[k].begin(), log.from_mask[k].end(), cap->from_mask + k * cells);
            if (cap->to_mask)
                std::copy(log.to_mask[k].begin(), log.to_mask[k].end(), cap->to_mask + k * cells);
        }
        if (cap->occupancy_k4)
            std::copy(st.occupancy.raw().begin(), st.occupancy.raw().end(), cap->occupancy_k4);
        if (cap->centers_k4) {
            for (std::size_t i = 0; i < peds; ++i) {
                cap->centers_k4[2 * i] = st.pedestrians[i].center.x;
                cap->centers_k4[2 * i + 1] = st.pedestrians[i].center.y;
            }
        }
    } else if (phase == 5) {
        if (cap->images_k5) {
            for (int k = 0; k < kDynKinds; ++k) {
                const auto& raw = st.dyn_images[k].raw();
                std::copy(raw.begin(), raw.end(), cap->images_k5 + k * cells * kSects);
            }
        }
    }
}

} // namespace

extern "C" {

const char* shim_impl_name(void) { return SHIM_IMPL_NAME; }

int shim_from_scenario(const char* text, int workers, shim_sim** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const ScenarioConfig cfg = parse_scenario(text);
        auto sim = std::make_unique<shim_sim>();
        sim->grid = cfg.grid;
        sim->ecfg = cfg.engine_config();
        sim->ecfg.workers = workers;
        sim->templates = cfg.field_templates();
        sim->state = seed_population(cfg);
        sim->engine = std::make_unique<Engine>(sim->grid, sim->ecfg, sim->templates);
        *out = sim.release();
    });
}

int shim_from_arrays(int width, int height, int closed, const shim_engine_cfg* cfg,
                     const shim_field templates[3], int64_t n, const int32_t* cx,
                     const int32_t* cy, const int32_t* fw, const int32_t* fh,
                     const int32_t* period, const int32_t* phase, const int32_t* goal,
                     shim_sim** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto sim = std::make_unique<shim_sim>();
        sim->grid = GridGeometry(width, height, closed ? BoundaryMode::Closed : BoundaryMode::Periodic);
        EngineConfig ec;
        ec.chunk_k = cfg->chunk_k;
        ec.weight_static = cfg->weight_static;
        ec.weight_dir_attractive = cfg->weight_dir_attractive;
        ec.weight_dir_repulsive = cfg->weight_dir_repulsive;
        ec.weight_recurrent = cfg->weight_recurrent;
        ec.goal_bias = cfg->goal_bias;
        ec.regulation = cfg->regulation == 0 ? Regulation::Identity : Regulation::Linear;
        ec.density_radius = cfg->density_radius;
        ec.rebuild_interval = static_cast<long>(cfg->rebuild_interval);
        ec.rebuild_tolerance = cfg->rebuild_tolerance;
        ec.workers = cfg->workers;
        ec.fault_invert_vote_tiebreak = cfg->fault_invert_vote_tiebreak != 0;
        sim->ecfg = ec;
        const FieldKind kinds[3] = {FieldKind::DirAttractive, FieldKind::DirRepulsive,
                                    FieldKind::RecurrentRepulsive};
        for (int k = 0; k < kDynKinds; ++k) {
            sim->templates[k] = FieldSpec(kinds[k], Footprint{templates[k].width, templates[k].height},
                                          templates[k].gain, templates[k].decay, 0);
        }
        SimState& st = sim->state;
        st.occupancy = OccupancyGrid(sim->grid);
        st.static_image = StrengthImage(sim->grid);
        st.pedestrians.reserve(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            Pedestrian p;
            p.id = static_cast<std::int32_t>(i);
            p.center = SuIndex{cx[i], cy[i]};
            p.footprint = Footprint{fw[i], fh[i]};
            p.walk_period = period[i];
            p.walk_phase = phase[i];
            p.goal_sect = goal[i];
            p.dyn_fields = sim->templates;
            for (auto& f : p.dyn_fields) {
                if (is_directional(f.kind)) f.orientation = p.goal_sect;
            }
            for (const SuIndex c : footprint_cells(sim->grid, p.center, p.footprint).cells) {
                st.occupancy.set(c, p.id);
            }
            st.pedestrians.push_back(std::move(p));
        }
        st.dyn_images = rasterize_dynamic(st.pedestrians, sim->grid);
        sim->engine = std::make_unique<Engine>(sim->grid, sim->ecfg, sim->templates);
        *out = sim.release();
    });
}

void shim_free(shim_sim* s) { delete s; }

int shim_set_static_fields(shim_sim* s, int64_t n, const shim_anchor* anchors, char* err,
                           size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<AnchoredField> fields;
        fields.reserve(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            const shim_anchor& a = anchors[i];
            const FieldKind kind = a.kind == 0 ? FieldKind::OmniAttractive : FieldKind::OmniRepulsive;
            fields.push_back(AnchoredField{FieldSpec(kind, Footprint{a.width, a.height}, a.gain, a.decay, 0),
                                           SuIndex{a.x, a.y}});
        }
        s->state.static_image = rasterize_static(fields, s->grid);
    });
}

int shim_grid(const shim_sim* s, int32_t* width, int32_t* height, int32_t* closed) {
    *width = s->grid.width;
    *height = s->grid.height;
    *closed = s->grid.boundary == BoundaryMode::Closed ? 1 : 0;
    return 0;
}

int64_t shim_population(const shim_sim* s) { return static_cast<int64_t>(s->state.pedestrians.size()); }
int64_t shim_tick_count(const shim_sim* s) { return s->state.tick; }
void shim_set_tick(shim_sim* s, int64_t tick) { s->state.tick = static_cast<long>(tick); }

int shim_run(shim_sim* s, int64_t ticks, int mode, int64_t* moved, int64_t* phase_us5, char* err,
             size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto metrics = s->engine->run(s->state, static_cast<long>(ticks), run_mode(mode));
        for (std::size_t i = 0; i < metrics.size(); ++i) {
            if (moved) moved[i] = metrics[i].moved;
            if (phase_us5)
                for (int p = 0; p < 5; ++p) phase_us5[i * 5 + p] = metrics[i].phase_us[p];
        }
    });
}

int shim_tick(shim_sim* s, int mode, int64_t* moved, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const TickMetrics m = s->engine->tick(s->state, run_mode(mode));
        if (moved) *moved = m.moved;
    });
}

int shim_tick_capture(shim_sim* s, int mode, shim_capture* cap, int64_t* moved, char* err,
                      size_t errlen) {
    return guarded(err, errlen, [&] {
        cap->phases_seen = 0;
        const TickMetrics m = s->engine->tick(
            s->state, run_mode(mode),
            [cap](int phase, const Engine& e, const SimState& st) { capture_phase(phase, e, st, cap); });
        if (moved) *moved = m.moved;
    });
}

int shim_verify(const shim_sim* s, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { s->engine->verify_state(s->state); });
}

int shim_decide(const shim_sim* s, int64_t ped, int32_t* direction, double* score, int32_t* ncells,
                int32_t* cells_xy, int32_t cap, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const MoveDecision d =
            s->engine->decide(s->state.pedestrians.at(static_cast<std::size_t>(ped)), s->state);
        *direction = d.direction;
        *score = d.score;
        *ncells = static_cast<int32_t>(d.new_cells.size());
        for (int32_t i = 0; i < *ncells && i < cap; ++i) {
            cells_xy[2 * i] = d.new_cells[static_cast<std::size_t>(i)].x;
            cells_xy[2 * i + 1] = d.new_cells[static_cast<std::size_t>(i)].y;
        }
    });
}

int shim_rebuild_images(const shim_sim* s, float* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto images = s->engine->rebuild_images(s->state);
        const std::size_t n = cell_count(s) * kSects;
        for (int k = 0; k < kDynKinds; ++k) {
            std::copy(images[k].raw().begin(), images[k].raw().end(), out + k * n);
        }
    });
}

int shim_plan_entries(const shim_sim* s, int kind, int orientation, int sect, int32_t* dxdy,
                      double* magnitude, int32_t cap) {
    const auto& entries = s->engine->plan(static_cast<DynKind>(kind), orientation).entries(sect);
    int32_t i = 0;
    for (const auto& e : entries) {
        if (i < cap) {
            if (dxdy) {
                dxdy[2 * i] = e.center_offset.dx;
                dxdy[2 * i + 1] = e.center_offset.dy;
            }
            if (magnitude) magnitude[i] = e.magnitude;
        }
        ++i;
    }
    return i;
}

int shim_plan_fanout(const shim_sim* s, int kind, int orientation) {
    return s->engine->plan(static_cast<DynKind>(kind), orientation).fanout();
}

void shim_get_centers(const shim_sim* s, int32_t* xy) {
    for (std::size_t i = 0; i < s->state.pedestrians.size(); ++i) {
        xy[2 * i] = s->state.pedestrians[i].center.x;
        xy[2 * i + 1] = s->state.pedestrians[i].center.y;
    }
}

void shim_get_ped_attrs(const shim_sim* s, int32_t* period, int32_t* phase, int32_t* goal,
                        int32_t* fw, int32_t* fh) {
    for (std::size_t i = 0; i < s->state.pedestrians.size(); ++i) {
        const Pedestrian& p = s->state.pedestrians[i];
        if (period) period[i] = p.walk_period;
        if (phase) phase[i] = p.walk_phase;
        if (goal) goal[i] = p.goal_sect;
        if (fw) fw[i] = p.footprint.width;
        if (fh) fh[i] = p.footprint.height;
    }
}

void shim_get_occupancy(const shim_sim* s, int32_t* out) {
    std::copy(s->state.occupancy.raw().begin(), s->state.occupancy.raw().end(), out);
}

void shim_get_image(const shim_sim* s, int which, float* out) {
    const StrengthImage& img = image_ref(const_cast<shim_sim*>(s), which);
    std::copy(img.raw().begin(), img.raw().end(), out);
}

void shim_set_centers(shim_sim* s, const int32_t* xy) {
    for (std::size_t i = 0; i < s->state.pedestrians.size(); ++i) {
        s->state.pedestrians[i].center = SuIndex{xy[2 * i], xy[2 * i + 1]};
    }
}

void shim_set_occupancy(shim_sim* s, const int32_t* in) {
    const int w = s->grid.width;
    for (std::size_t i = 0; i < cell_count(s); ++i) {
        s->state.occupancy.set(SuIndex{static_cast<int>(i % w), static_cast<int>(i / w)}, in[i]);
    }
}

void shim_set_image(shim_sim* s, int which, const float* in) {
    StrengthImage& img = image_ref(s, which);
    const int w = s->grid.width;
    for (std::size_t i = 0; i < cell_count(s); ++i) {
        const SuIndex su{static_cast<int>(i % w), static_cast<int>(i / w)};
        for (int sect = 0; sect < kSects; ++sect) img.at(su, sect) = in[i * kSects + sect];
    }
}

uint64_t shim_digest(const shim_sim* s) {
    std::uint64_t h = 14695981039346656037ull;
    const auto& occ = s->state.occupancy.raw();
    h = fnv1a(occ.data(), occ.size() * sizeof(std::int32_t), h);
    for (const auto& img : s->state.dyn_images) {
        h = fnv1a(img.raw().data(), img.raw().size() * sizeof(float), h);
    }
    for (const auto& p : s->state.pedestrians) {
        const std::int32_t xy[2] = {p.center.x, p.center.y};
        h = fnv1a(xy, sizeof xy, h);
    }
    return h;
}

int shim_states_identical(const shim_sim* a, const shim_sim* b, char* diag, size_t diaglen) {
    std::string why;
    const bool same = states_identical(a->state, b->state, &why);
    if (!same) put_err(diag, diaglen, why);
    return same ? 1 : 0;
}

int shim_clone(const shim_sim* s, shim_sim** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto sim = std::make_unique<shim_sim>();
        sim->grid = s->grid;
        sim->ecfg = s->ecfg;
        sim->templates = s->templates;
        sim->state = s->state;
        sim->engine = std::make_unique<Engine>(sim->grid, sim->ecfg, sim->templates);
        *out = sim.release();
    });
}

int shim_sect_index(double x, double y) { return sect_index(x, y); }

void shim_sort8_desc(const double scores[8], int32_t order[8]) {
    std::array<double, 8> in;
    std::copy(scores, scores + 8, in.begin());
    const auto o = sort8_desc(in);
    for (int i = 0; i < 8; ++i) order[i] = o[static_cast<std::size_t>(i)];
}

double shim_multi_step_sum(const double* terms, int64_t n, int k) {
    return multi_step_sum(std::span<const double>(terms, static_cast<std::size_t>(n)), k);
}

void shim_strength_at_offset(int kind, int w, int h, double gain, double decay, int orientation,
                             int dx, int dy, double* sx, double* sy) {
    const FieldSpec f(static_cast<FieldKind>(kind), Footprint{w, h}, gain, decay, orientation);
    const Vec2 v = strength_at_offset(f, Offset{dx, dy});
    *sx = v.x;
    *sy = v.y;
}

} // extern "C"
