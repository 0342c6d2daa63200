// evr_resident.cuh -- persistent on-chip engine (placeholder: never fits)
#pragma once
struct evr_ctx;
namespace evr {
struct ResidentPlan { int ctas = 0; };
template <class T> bool resident_plan(evr_ctx*, ResidentPlan&) { return false; }
template <class T> int resident_alloc(evr_ctx*) { return 0; }
template <class T> int resident_enqueue(evr_ctx*, int) { return -5; }
}  // namespace evr
