// store.h — device-resident CoefficientStore (see store.cu)
#pragma once

#include <cstddef>
#include <memory>

namespace qapb {

size_t store_nb(int m);
size_t store_nc(int m);
size_t store_nd(int m);

// b, c, d in the reference layout (StoreIndex, rlt2.hpp:25-69), in HBM
struct DeviceStore {
  int m = 0;
  int device = 0;
  double* b = nullptr;
  double* c = nullptr;
  double* d = nullptr;
  double offset = 0.0;
  DeviceStore(int m_, int device_);
  ~DeviceStore();
  DeviceStore(const DeviceStore&) = delete;
  DeviceStore& operator=(const DeviceStore&) = delete;
};

// collapse_store, rlt2.cpp:109-182, bitwise, on the store's device
std::unique_ptr<DeviceStore> collapse_store_device(const DeviceStore& s, int fac, int loc);

}  // namespace qapb
